"""pkgpu — B200-native periodic KIFMM evaluator (drop-in for pkifmm::evaluate).

Python mirror of the reference's public C++ interface (include/pkifmm/fmm.hpp,
geometry.hpp, kernel.hpp, periodize.hpp) over the C ABI in include/pkgpu.h. Names,
argument meaning and error classes follow the reference:

    std::invalid_argument   -> ValueError
    pkifmm::ConfigError     -> ConfigError
    std::runtime_error      -> RuntimeError (CudaError for device failures)

All compute runs in libpkgpu.so (hand-written sm_100a CUDA). There is no CPU fallback:
importing works without a GPU (for the build check), but every compute call needs the
extension and a CUDA device and fails loudly otherwise.
"""
from __future__ import annotations

import ctypes
import enum
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

__all__ = [
    "KernelType", "KernelSpec", "Periodicity", "PeriodicSetup", "EvalMode", "EvalRequest", "EvalResult",
    "EvalTimings", "CompatReport", "PeriodizingOperator", "ConfigError", "CudaError", "Context", "FmmTree",
    "evaluate", "load_operator", "kernel_block_apply", "surface_points", "surface_point_count", "generate",
    "set_kifmm_factors", "get_kifmm_factors", "kifmm_matrix", "crc64", "lib", "LIB_PATH", "TorchDistComm",
    "ThreadComm",
]

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpkgpu.so")


class ConfigError(RuntimeError):
    """pkifmm::ConfigError (include/pkifmm/refsum.hpp:16-18)."""


class CudaError(RuntimeError):
    """Device failure inside libpkgpu."""


# ---------------------------------------------------------------------------
# C ABI binding

class _Setup(ctypes.Structure):
    _fields_ = [("periodicity", ctypes.c_int), ("axes", ctypes.c_int * 3), ("box_length", ctypes.c_double),
                ("ell", ctypes.c_int)]


class _Request(ctypes.Structure):
    _fields_ = [("kernel", ctypes.c_int), ("n_sources", ctypes.c_int64), ("sources", ctypes.c_void_p),
                ("n_strengths", ctypes.c_int64), ("strengths", ctypes.c_void_p), ("n_targets", ctypes.c_int64),
                ("targets", ctypes.c_void_p), ("setup", _Setup), ("p", ctypes.c_int), ("op", ctypes.c_void_p),
                ("mode", ctypes.c_int), ("leaf_capacity", ctypes.c_int), ("force", ctypes.c_int),
                ("device_pointers", ctypes.c_int)]


_ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t)
_ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p)
_ALLTOALLV_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64),
                                 ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p)
_ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p)


class _Partition(ctypes.Structure):
    """pkgpu_partition (include/pkgpu.h): rank, nranks, alloc, allreduce, user, and the
    optional alltoallv (halo exchange) and allgather (small-level int8 run by modulus)."""
    _fields_ = [("rank", ctypes.c_int), ("nranks", ctypes.c_int), ("alloc", _ALLOC_FN),
                ("allreduce", _ALLREDUCE_FN), ("user", ctypes.c_void_p), ("alltoallv", _ALLTOALLV_FN),
                ("allgather", _ALLGATHER_FN)]


class _Timings(ctypes.Structure):
    _fields_ = [("tree", ctypes.c_double), ("near", ctypes.c_double), ("m2l_apply", ctypes.c_double),
                ("far", ctypes.c_double)]


class _Ewald(ctypes.Structure):
    _fields_ = [("xi", ctypes.c_double), ("real_shells", ctypes.c_int), ("wave_cutoff", ctypes.c_int),
                ("n_images", ctypes.c_longlong)]


class _Compat(ctypes.Structure):
    _fields_ = [("ok", ctypes.c_int), ("residual", ctypes.c_double), ("violated", ctypes.c_char * 96)]


_lib = None
P = ctypes.c_void_p
D = ctypes.POINTER(ctypes.c_double)
I64 = ctypes.c_int64
ERR = ctypes.c_char_p
SZ = ctypes.c_size_t

_SIGNATURES = {
    "pkgpu_context_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(P), ERR, SZ]),
    "pkgpu_context_destroy": (None, [P]),
    "pkgpu_context_set_stream": (ctypes.c_int, [P, P]),
    "pkgpu_context_stream": (P, [P]),
    "pkgpu_context_launch_count": (I64, [P]),
    "pkgpu_context_set_profiling": (ctypes.c_int, [P, ctypes.c_int]),
    "pkgpu_context_reset_stats": (ctypes.c_int, [P]),
    "pkgpu_context_set_m2l": (ctypes.c_int, [P, ctypes.c_int, I64, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "pkgpu_i8_gather_gemm": (ctypes.c_int, [P, P, ctypes.c_int, P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                            ctypes.c_int, P, I64, I64, ctypes.c_int, ctypes.c_int, P, ERR, SZ]),
    "pkgpu_i8_moduli": (ctypes.c_int, [P, ctypes.c_int]),
    "pkgpu_context_stage_stats": (ctypes.c_int, [P, ctypes.c_char_p, ctypes.POINTER(ctypes.c_double),
                                                 ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                                 ctypes.POINTER(I64)]),
    "pkgpu_evaluate": (ctypes.c_int, [P, ctypes.POINTER(_Request), P, ctypes.POINTER(_Timings),
                                      ctypes.POINTER(_Compat), ERR, SZ]),
    "pkgpu_evaluate_partitioned": (ctypes.c_int, [P, ctypes.POINTER(_Request), P, P, ctypes.POINTER(_Timings),
                                                  ctypes.POINTER(_Compat), ERR, SZ]),
    "pkgpu_operator_load": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(P), ERR, SZ]),
    "pkgpu_operator_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_Setup), ctypes.c_int, P, I64,
                                             ctypes.POINTER(P), ERR, SZ]),
    "pkgpu_operator_free": (None, [P]),
    "pkgpu_operator_info": (ctypes.c_int, [P, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(_Setup),
                                           ctypes.POINTER(ctypes.c_int), ctypes.POINTER(I64),
                                           ctypes.POINTER(ctypes.c_double)]),
    "pkgpu_operator_relabel": (ctypes.c_int, [P, ctypes.c_int, ctypes.POINTER(_Setup)]),
    "pkgpu_operator_matrix": (ctypes.c_int, [P, P]),
    "pkgpu_crc64": (ctypes.c_uint64, [P, SZ]),
    "pkgpu_operator_solve": (ctypes.c_int, [P, ctypes.c_int, ctypes.POINTER(_Setup), ctypes.c_int,
                                            ctypes.POINTER(_Ewald), ctypes.c_int, ctypes.POINTER(P), ERR, SZ]),
    "pkgpu_operator_save": (ctypes.c_int, [P, ctypes.c_char_p, ERR, SZ]),
    "pkgpu_periodic_block": (ctypes.c_int, [P, ctypes.c_int, ctypes.POINTER(_Setup), ctypes.POINTER(_Ewald),
                                            ctypes.c_int, P, I64, P, I64, P, ERR, SZ]),
    "pkgpu_oracle_system_eval": (ctypes.c_int, [P, ctypes.c_int, ctypes.POINTER(_Setup), ctypes.POINTER(_Ewald), P,
                                                I64, P, P, I64, P, ERR, SZ]),
    "pkgpu_set_kifmm_factors": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, P, P, P, P, P, P, ERR, SZ]),
    "pkgpu_get_kifmm_factors": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, P, P, P, P, P, P, ERR, SZ]),
    "pkgpu_kifmm_matrix": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_int, P, ERR, SZ]),
    "pkgpu_kernel_block_apply": (ctypes.c_int, [P, ctypes.c_int, P, I64, P, I64, P, P, P, ctypes.c_int, ERR, SZ]),
    "pkgpu_surface_points": (ctypes.c_int, [ctypes.c_int, P, ctypes.c_double, P]),
    "pkgpu_tree_build": (ctypes.c_int, [P, P, I64, P, I64, ctypes.c_int, ctypes.POINTER(P), ERR, SZ]),
    "pkgpu_tree_free": (None, [P]),
    "pkgpu_tree_info": (ctypes.c_int, [P, ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(ctypes.c_int),
                                       ctypes.POINTER(ctypes.c_uint64)]),
    "pkgpu_tree_boxes": (ctypes.c_int, [P, P, P, P]),
    "pkgpu_tree_lists": (ctypes.c_int, [P, ctypes.POINTER(_Setup), ctypes.c_int, P, P, ERR, SZ]),
    "pkgpu_generate": (ctypes.c_int, [ctypes.c_int, I64, ctypes.c_int, ctypes.c_double, ctypes.POINTER(ctypes.c_int),
                                      ctypes.c_int, ctypes.c_uint64, P, P]),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)


def lib():
    """The loaded libpkgpu.so (raises if the extension is not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libpkgpu.so not built ({LIB_PATH}); run `python -c 'import __graft_entry__ as g; "
                              "g.build()'` (no CPU fallback exists)")
        l = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(l, name)
            fn.restype = res
            fn.argtypes = args
        _lib = l
    return _lib


_STATUS = {1: ValueError, 2: ConfigError, 3: RuntimeError, 4: CudaError}


def _check(status, err):
    if status != 0:
        msg = err.value.decode(errors="replace") if err is not None else ""
        raise _STATUS.get(status, RuntimeError)(msg)


def _errbuf():
    return ctypes.create_string_buffer(1024)


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None and a.size else ctypes.c_void_p(0)


# ---------------------------------------------------------------------------
# reference types (include/pkifmm/kernel.hpp, geometry.hpp)

class KernelType(enum.IntEnum):
    laplace = 0
    stokeslet = 1


@dataclass(frozen=True)
class KernelSpec:
    """Laplace 1/|r| (no 1/4pi) or the Stokeslet (1/8pi)(I/|r| + r r^T/|r|^3)."""
    type: KernelType = KernelType.laplace

    @property
    def ks(self):
        return 1 if self.type == KernelType.laplace else 3

    @property
    def kt(self):
        return self.ks

    @staticmethod
    def laplace():
        return KernelSpec(KernelType.laplace)

    @staticmethod
    def stokeslet():
        return KernelSpec(KernelType.stokeslet)

    @staticmethod
    def from_name(name):
        if name == "laplace":
            return KernelSpec.laplace()
        if name in ("stokeslet", "stokes"):
            return KernelSpec.stokeslet()
        raise ValueError(f"unknown kernel name: {name}")

    def name(self):
        return "laplace" if self.type == KernelType.laplace else "stokeslet"


class Periodicity(enum.IntEnum):
    none = 0
    sp = 1
    dp = 2
    tp = 3

    @staticmethod
    def from_name(name):
        try:
            return Periodicity[name]
        except KeyError:
            raise ValueError(f"unknown periodicity: {name}") from None


@dataclass
class PeriodicSetup:
    periodicity: Periodicity = Periodicity.none
    axes: tuple = (False, False, False)
    box_length: float = 1.0
    ell: int = 2

    @staticmethod
    def make(periodicity, ell=2):
        """PeriodicSetup::make (src/geometry.cpp:27-39): SP along z, DP in x-y, TP all."""
        if ell < 1:
            raise ValueError("PeriodicSetup: ell must be >= 1")
        periodicity = Periodicity(periodicity)
        axes = {Periodicity.none: (False, False, False), Periodicity.sp: (False, False, True),
                Periodicity.dp: (True, True, False), Periodicity.tp: (True, True, True)}[periodicity]
        return PeriodicSetup(periodicity, axes, 1.0, ell)

    def dim(self):
        return sum(bool(a) for a in self.axes)

    def _c(self):
        s = _Setup()
        s.periodicity = int(self.periodicity)
        for i in range(3):
            s.axes[i] = 1 if self.axes[i] else 0
        s.box_length = self.box_length
        s.ell = self.ell
        return s

    @staticmethod
    def _from_c(s):
        return PeriodicSetup(Periodicity(s.periodicity), tuple(bool(s.axes[i]) for i in range(3)), s.box_length,
                             s.ell)


class EvalMode(enum.IntEnum):
    fmm = 0
    direct = 1


@dataclass
class EvalTimings:
    tree: float = 0.0
    near: float = 0.0
    m2l_apply: float = 0.0
    far: float = 0.0


@dataclass
class CompatReport:
    ok: bool = True
    violated: str = ""
    residual: float = 0.0


@dataclass
class EvalResult:
    potentials: object
    timings: EvalTimings
    compat: CompatReport


def surface_point_count(p):
    return 6 * (p - 1) * (p - 1) + 2


class PeriodizingOperator:
    """The dense periodizing operator T_M2L with its provenance
    (include/pkifmm/periodize.hpp:22-33). Owns a pkgpu_operator handle."""

    def __init__(self, handle):
        self._h = ctypes.c_void_p(handle)

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value and _lib is not None:
            _lib.pkgpu_operator_free(self._h)
            self._h = ctypes.c_void_p(0)

    def _info(self):
        k, s, p, dim, res = ctypes.c_int(), _Setup(), ctypes.c_int(), ctypes.c_int64(), ctypes.c_double()
        lib().pkgpu_operator_info(self._h, ctypes.byref(k), ctypes.byref(s), ctypes.byref(p), ctypes.byref(dim),
                                  ctypes.byref(res))
        return KernelSpec(KernelType(k.value)), PeriodicSetup._from_c(s), p.value, dim.value, res.value

    @property
    def kernel(self):
        return self._info()[0]

    @property
    def setup(self):
        return self._info()[1]

    @property
    def p(self):
        return self._info()[2]

    @property
    def residual_max(self):
        return self._info()[4]

    @property
    def matrix(self):
        dim = self._info()[3]
        m = np.empty((dim, dim))
        lib().pkgpu_operator_matrix(self._h, _ptr(m))
        return m

    def relabel(self, kernel: KernelSpec, setup: PeriodicSetup):
        """Overwrite the provenance (SP-x permuted operator, DP-Stokes stand-in)."""
        s = setup._c()
        if lib().pkgpu_operator_relabel(self._h, int(kernel.type), ctypes.byref(s)) != 0:
            raise ValueError("relabel: kernel dimension does not match the operator")
        return self

    @staticmethod
    def create(kernel: KernelSpec, setup: PeriodicSetup, p: int, matrix):
        m = np.ascontiguousarray(matrix, dtype=np.float64)
        h, err, s = ctypes.c_void_p(), _errbuf(), setup._c()
        _check(lib().pkgpu_operator_create(int(kernel.type), ctypes.byref(s), p, _ptr(m), m.shape[0],
                                           ctypes.byref(h), err, 1024), err)
        return PeriodizingOperator(h.value)


class EwaldParams:
    """EwaldParams (include/pkifmm/refsum.hpp:21-27)."""

    def __init__(self, xi=8.0, real_shells=2, wave_cutoff=64, n_images=1_000_000):
        self.xi, self.real_shells, self.wave_cutoff, self.n_images = xi, real_shells, wave_cutoff, n_images

    def _c(self):
        return _Ewald(float(self.xi), int(self.real_shells), int(self.wave_cutoff), int(self.n_images))


def solve_m2l(kernel: KernelSpec, setup: PeriodicSetup, p: int, params: Optional[EwaldParams] = None,
              gated: bool = True, context: Optional["Context"] = None) -> PeriodizingOperator:
    """solve_m2l (include/pkifmm/periodize.hpp:42) on the GPU: K^{P,F} on the inner root
    surface, T = pinv(a_dn) K^{P,F}, backward-residual gate 1e-11 (gated=False: the ungated
    operator, residual_max = -1). ConfigError for unsupported (kernel, periodicity)."""
    ctx = context or default_context()
    h, err, s, e = ctypes.c_void_p(), _errbuf(), setup._c(), (params or EwaldParams())._c()
    _check(lib().pkgpu_operator_solve(ctx._h, int(kernel.type), ctypes.byref(s), int(p), ctypes.byref(e),
                                      1 if gated else 0, ctypes.byref(h), err, 1024), err)
    return PeriodizingOperator(h.value)


def save_operator(op: PeriodizingOperator, path) -> None:
    """save_operator (include/pkifmm/periodize.hpp:61): PKM2L with the reference's header."""
    err = _errbuf()
    _check(lib().pkgpu_operator_save(op._h, str(path).encode(), err, 1024), err)


def periodic_block(kernel: KernelSpec, setup: PeriodicSetup, targets, sources, far_only=False,
                   params: Optional[EwaldParams] = None, context: Optional["Context"] = None):
    """periodic_block / kpf_block (include/pkifmm/refsum.hpp:68-72) on the GPU."""
    ctx = context or default_context()
    t = np.ascontiguousarray(targets, dtype=np.float64).reshape(-1, 3)
    sr = np.ascontiguousarray(sources, dtype=np.float64).reshape(-1, 3)
    k = kernel.ks
    out = np.empty((k * len(t), k * len(sr)))
    err, s, e = _errbuf(), setup._c(), (params or EwaldParams())._c()
    _check(lib().pkgpu_periodic_block(ctx._h, int(kernel.type), ctypes.byref(s), ctypes.byref(e),
                                      1 if far_only else 0, _ptr(t), len(t), _ptr(sr), len(sr), _ptr(out), err,
                                      1024), err)
    return out


def oracle_system_eval(kernel: KernelSpec, setup: PeriodicSetup, sources, strengths, targets,
                       params: Optional[EwaldParams] = None, context: Optional["Context"] = None):
    """oracle_system_eval (include/pkifmm/refsum.hpp:88): q_t = sum_s K^P(x_t, y_s) phi_s."""
    ctx = context or default_context()
    sr = np.ascontiguousarray(sources, dtype=np.float64).reshape(-1, 3)
    q = np.ascontiguousarray(strengths, dtype=np.float64).reshape(-1)
    t = np.ascontiguousarray(targets, dtype=np.float64).reshape(-1, 3)
    out = np.empty(kernel.kt * len(t))
    err, s, e = _errbuf(), setup._c(), (params or EwaldParams())._c()
    _check(lib().pkgpu_oracle_system_eval(ctx._h, int(kernel.type), ctypes.byref(s), ctypes.byref(e), _ptr(sr),
                                          len(sr), _ptr(q), _ptr(t), len(t), _ptr(out), err, 1024), err)
    return out


def load_operator(path) -> PeriodizingOperator:
    """load_operator (src/periodize.cpp:231-278): PKM2L magic, header, CRC-64/XZ."""
    h, err = ctypes.c_void_p(), _errbuf()
    _check(lib().pkgpu_operator_load(str(path).encode(), ctypes.byref(h), err, 1024), err)
    return PeriodizingOperator(h.value)


def crc64(data: bytes) -> int:
    buf = ctypes.create_string_buffer(bytes(data), len(data))
    return lib().pkgpu_crc64(ctypes.cast(buf, ctypes.c_void_p), len(data))


# ---------------------------------------------------------------------------
# context

class Context:
    """Device, stream and device-resident operator caches (the reference's static
    registries, src/fmm.cpp:238-283)."""

    def __init__(self, device=0):
        h, err = ctypes.c_void_p(), _errbuf()
        _check(lib().pkgpu_context_create(device, ctypes.byref(h), err, 1024), err)
        self._h = h
        self.device = device
        self._explicit_stream = False

    def close(self):
        if self._h and self._h.value:
            lib().pkgpu_context_destroy(self._h)
            self._h = ctypes.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: int):
        """Run this context's work on `stream_ptr` (a cudaStream_t; 0 = the context's own
        stream). Without an explicit stream, device-resident evaluates run on torch's
        current stream of the inputs' device (see evaluate)."""
        lib().pkgpu_context_set_stream(self._h, ctypes.c_void_p(stream_ptr))
        self._explicit_stream = True

    @property
    def stream(self) -> int:
        return lib().pkgpu_context_stream(self._h) or 0

    @property
    def launches(self) -> int:
        return lib().pkgpu_context_launch_count(self._h)

    STAGES = ("tree", "lists", "s2m", "m2m", "pinv_up", "x", "m2l", "l2l", "pinv_dn", "periodic", "leaf",
              "m2l_prep", "m2l_i8", "m2l_crt",  # sub-stages of m2l on the int8 pipe
              "lat_fwd", "lat_mul", "lat_inv")  # sub-stages of m2l on the lattice path (lat_mul "flops" = bytes)

    def set_profiling(self, on: bool):
        lib().pkgpu_context_set_profiling(self._h, 1 if on else 0)

    def set_m2l(self, path="int8", min_boxes=0, nmod=0, beta_a=0, beta_b=0):
        """M2L arithmetic: "int8" (exact residue GEMMs on the int8 tensor pipe for levels
        with >= min_boxes boxes, FP64 DMMA elsewhere; the default) or "dmma" (FP64 DMMA
        everywhere) or "int8_all" (as "int8", plus M2M / L2L / pseudo-inverses on the int8
        pipe) or "fft" (FP64 FFT convolution on the surface lattice, the PVFMM scheme) or
        "int8_dense" (as "int8" without the lattice FFT M2L). Except with "dmma" and
        "int8_dense", levels whose box lattice is filled run M2L as one convolution over the
        lattice (surface FFT x lattice FFT, FP64; PKGPU_M2L_LATTICE=0 disables it).
        nmod / beta_a / beta_b override the residue parameters."""
        code = {"int8": 0, "dmma": 1, "int8_all": 2, "fft": 3, "int8_dense": 4}[path]
        if lib().pkgpu_context_set_m2l(self._h, code, int(min_boxes), int(nmod), int(beta_a), int(beta_b)) != 0:
            raise ValueError(f"set_m2l: invalid settings {path, min_boxes, nmod, beta_a, beta_b}")

    def reset_stats(self):
        lib().pkgpu_context_reset_stats(self._h)

    def stage_stats(self):
        """{stage: dict(seconds, units, flops, launches)} accumulated while profiling."""
        out = {}
        for st in self.STAGES + ("u_pairs", "m2l_mma_rows", "m2l_lattice", "dmma_gemm"):
            sec, un, fl, ln = ctypes.c_double(), ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
            if lib().pkgpu_context_stage_stats(self._h, st.encode(), ctypes.byref(sec), ctypes.byref(un),
                                               ctypes.byref(fl), ctypes.byref(ln)) == 0:
                out[st] = dict(seconds=sec.value, units=un.value, flops=fl.value, launches=ln.value)
        return out


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


# ---------------------------------------------------------------------------
# evaluate

@dataclass
class EvalRequest:
    """EvalRequest (include/pkifmm/fmm.hpp:120-131). sources/targets: (N, 3) float64
    (numpy, or torch CUDA tensors for the device-resident path); strengths: ks per source."""
    kernel: KernelSpec = field(default_factory=KernelSpec.laplace)
    sources: object = None
    strengths: object = None
    targets: object = None
    setup: PeriodicSetup = field(default_factory=PeriodicSetup)
    p: int = 8
    op: Optional[PeriodizingOperator] = None
    mode: EvalMode = EvalMode.fmm
    leaf_capacity: int = 1000
    force: bool = False


def _is_torch_cuda(x):
    return hasattr(x, "is_cuda") and getattr(x, "is_cuda")


def evaluate(request: EvalRequest, context: Optional[Context] = None, out=None, comm=None) -> EvalResult:
    """pkifmm::evaluate (src/fmm.cpp:690-742): near field over ell image layers + far
    field through the periodizing operator, on the GPU.

    comm: optional communicator (TorchDistComm / ThreadComm) -> Morton-range partitioned
    evaluation across ranks (pkgpu_evaluate_partitioned); every rank passes the full
    request and receives the full potentials."""
    ctx = context or default_context()
    k = request.kernel
    dev = _is_torch_cuda(request.sources)
    r = _Request()
    r.kernel = int(k.type)
    r.setup = request.setup._c()
    r.p = int(request.p)
    r.op = request.op._h if request.op is not None else None
    r.mode = int(request.mode)
    r.leaf_capacity = int(request.leaf_capacity)
    r.force = 1 if request.force else 0
    r.device_pointers = 1 if dev else 0
    if dev:
        import torch
        src, q, trg = request.sources, request.strengths, request.targets
        for name, t in (("sources", src), ("strengths", q), ("targets", trg)):
            if not _is_torch_cuda(t) or t.device.index != ctx.device:
                raise ValueError(f"{name}: device inputs must all be CUDA tensors on the context's device "
                                 f"cuda:{ctx.device}")
            if not (t.is_contiguous() and t.dtype == torch.float64):
                raise ValueError(f"{name}: device inputs must be contiguous float64 CUDA tensors")
        if src.numel() % 3 or trg.numel() % 3:
            raise ValueError("sources / targets: xyz triples expected (numel divisible by 3)")
        ns, nq, nt = src.numel() // 3, q.numel(), trg.numel() // 3
        r.sources, r.strengths, r.targets = src.data_ptr(), q.data_ptr(), trg.data_ptr()
        if out is None:
            out = torch.empty(k.kt * nt, dtype=torch.float64, device=src.device)
        elif not (_is_torch_cuda(out) and out.device.index == ctx.device and out.dtype == torch.float64
                  and out.is_contiguous() and out.numel() == k.kt * nt):
            raise ValueError(f"out: a contiguous float64 CUDA tensor on cuda:{ctx.device} with {k.kt * nt} "
                             "elements is required")
        # stream contract: without an explicit context stream the evaluate runs on torch's
        # current stream, ordered after the kernels / copies that produced the inputs
        if not ctx._explicit_stream:
            lib().pkgpu_context_set_stream(ctx._h, ctypes.c_void_p(torch.cuda.current_stream(src.device).cuda_stream))
        optr = out.data_ptr()
    else:
        for name, t in (("strengths", request.strengths), ("targets", request.targets)):
            if _is_torch_cuda(t):
                raise ValueError(f"{name}: mixed host and device inputs")
        src = np.ascontiguousarray(request.sources, dtype=np.float64).reshape(-1, 3)
        q = np.ascontiguousarray(request.strengths, dtype=np.float64).reshape(-1)
        trg = np.ascontiguousarray(request.targets, dtype=np.float64).reshape(-1, 3)
        ns, nq, nt = len(src), q.size, len(trg)
        r.sources, r.strengths, r.targets = _ptr(src), _ptr(q), _ptr(trg)
        if out is None:
            out = np.zeros(k.kt * nt)
        elif not (isinstance(out, np.ndarray) and out.dtype == np.float64 and out.flags.c_contiguous
                  and out.size == k.kt * nt):
            raise ValueError(f"out: a C-contiguous float64 numpy array with {k.kt * nt} elements is required")
        optr = out.ctypes.data
    r.n_sources, r.n_strengths, r.n_targets = ns, nq, nt
    tm, cp, err = _Timings(), _Compat(), _errbuf()
    if comm is not None and comm.nranks > 1:
        comm.begin_call()
        part = _Partition(comm.rank, comm.nranks, comm.c_alloc, comm.c_allreduce, None, comm.c_alltoallv,
                          comm.c_allgather)
        try:
            st = lib().pkgpu_evaluate_partitioned(ctx._h, ctypes.byref(r), ctypes.byref(part), ctypes.c_void_p(optr),
                                                  ctypes.byref(tm), ctypes.byref(cp), err, 1024)
        finally:
            comm.end_call()
        if comm.error is not None:
            raise comm.error
        _check(st, err)
    else:
        _check(lib().pkgpu_evaluate(ctx._h, ctypes.byref(r), ctypes.c_void_p(optr), ctypes.byref(tm),
                                    ctypes.byref(cp), err, 1024), err)
    return EvalResult(out, EvalTimings(tm.tree, tm.near, tm.m2l_apply, tm.far),
                      CompatReport(bool(cp.ok), cp.violated.decode(), cp.residual))


# ---------------------------------------------------------------------------
# communicators for the partitioned path (pkgpu_evaluate_partitioned)

class _CommBase:
    """Supplies the two callbacks of pkgpu_partition: device allocation (torch tensors, so
    the collective can run on them) and an in-place sum over ranks."""

    def __init__(self, rank, nranks, device=0):
        self.rank, self.nranks, self.device = rank, nranks, device
        self._bufs = {}
        self.error = None
        self.c_alloc = _ALLOC_FN(self._alloc)
        self.c_allreduce = _ALLREDUCE_FN(self._allreduce)
        # the halo / modulus-split collectives; set_v1() reverts to round 1's single allreduce
        self.c_alltoallv = _ALLTOALLV_FN(self._alltoallv)
        self.c_allgather = _ALLGATHER_FN(self._allgather)
        self.moved = 0  # doubles this rank received through the collectives (last call)

    def set_v1(self):
        """Exchange every box's equivalent density with one allreduce (no halo exchange,
        no modulus split): the library falls back when the optional callbacks are NULL."""
        self.c_alltoallv = _ALLTOALLV_FN()
        self.c_allgather = _ALLGATHER_FN()

    def begin_call(self):
        self._bufs.clear()
        self.error = None
        self.moved = 0

    def end_call(self):
        self._bufs.clear()

    def _alloc(self, user, nbytes):
        try:
            import torch
            dev = torch.device("cpu") if self.device == "cpu" else torch.device("cuda", self.device)
            t = torch.empty(max(1, (nbytes + 7) // 8), dtype=torch.float64, device=dev)
            self._bufs[t.data_ptr()] = t
            return t.data_ptr()
        except Exception as e:  # never let an exception cross the C boundary
            self.error = e
            return None

    def _find(self, ptr, count):
        """The allocated tensor holding [ptr, ptr + count doubles) as a view."""
        for base, t in self._bufs.items():
            if base <= ptr and ptr + 8 * count <= base + 8 * t.numel():
                o = (ptr - base) // 8
                return t[o:o + count]
        raise KeyError("pkgpu: collective on memory not from the alloc callback")

    def _allreduce(self, user, ptr, count, stream):
        try:
            self.allreduce(self._find(ptr, count))
            self.moved += count
            return 0
        except Exception as e:
            self.error = e
            return 1

    def _alltoallv(self, user, sptr, scounts, rptr, rcounts, stream):
        try:
            sc = [int(scounts[q]) for q in range(self.nranks)]
            rc = [int(rcounts[q]) for q in range(self.nranks)]
            self.alltoallv(self._find(sptr, max(1, sum(sc)))[:sum(sc)], sc, self._find(rptr, max(1, sum(rc)))[:sum(rc)],
                           rc)
            self.moved += sum(rc)
            return 0
        except Exception as e:
            self.error = e
            return 1

    def _allgather(self, user, ptr, nbytes, stream):
        try:
            n = (nbytes + 7) // 8
            self.allgather(self._find(ptr, n * self.nranks), n)
            self.moved += n * (self.nranks - 1)
            return 0
        except Exception as e:
            self.error = e
            return 1

    def allreduce(self, t):
        raise NotImplementedError

    def alltoallv(self, send, send_counts, recv, recv_counts):
        raise NotImplementedError

    def allgather(self, buf, n):
        raise NotImplementedError


class TorchDistComm(_CommBase):
    """torch.distributed (NCCL over NVLink on the GPU box) communicator."""

    def __init__(self, group=None, device=None):
        import torch.distributed as dist
        rank, n = dist.get_rank(group), dist.get_world_size(group)
        super().__init__(rank, n, device if device is not None else int(os.environ.get("LOCAL_RANK", "0")))
        self.group = group

    def allreduce(self, t):
        import torch
        import torch.distributed as dist
        dist.all_reduce(t, group=self.group)
        if t.is_cuda:
            torch.cuda.synchronize(t.device)

    def alltoallv(self, send, send_counts, recv, recv_counts):
        import torch
        import torch.distributed as dist
        dist.all_to_all_single(recv, send, output_split_sizes=recv_counts, input_split_sizes=send_counts,
                               group=self.group)
        if recv.is_cuda:
            torch.cuda.synchronize(recv.device)

    def allgather(self, buf, n):
        import torch
        import torch.distributed as dist
        mine = buf[self.rank * n:(self.rank + 1) * n].clone()
        dist.all_gather_into_tensor(buf, mine, group=self.group)
        if buf.is_cuda:
            torch.cuda.synchronize(buf.device)


class ThreadComm:
    """In-process emulation of R ranks as host threads sharing one GPU (tests): the sum
    runs between host barriers, no kernel ever waits on another rank's kernel."""

    def __init__(self, nranks, device=0):
        import threading
        self.nranks, self.device = nranks, device
        self.barrier = threading.Barrier(nranks)
        self.slots = [None] * nranks
        self.result = None

    def rank(self, r):
        outer = self

        class _Rank(_CommBase):
            def allreduce(self, t):
                import torch
                torch.cuda.synchronize()
                outer.slots[r] = t
                outer.barrier.wait()
                if r == 0:
                    acc = outer.slots[0].clone()
                    for s in outer.slots[1:]:
                        acc += s
                    outer.result = acc
                    torch.cuda.synchronize()
                outer.barrier.wait()
                t.copy_(outer.result)
                torch.cuda.synchronize()
                outer.barrier.wait()

            def alltoallv(self, send, send_counts, recv, recv_counts):
                import torch
                torch.cuda.synchronize()
                outer.slots[r] = (send, send_counts)
                outer.barrier.wait()
                o = 0
                for q in range(outer.nranks):
                    s_q, c_q = outer.slots[q]
                    off = sum(c_q[:r])
                    assert c_q[r] == recv_counts[q]
                    recv[o:o + recv_counts[q]].copy_(s_q[off:off + c_q[r]])
                    o += recv_counts[q]
                torch.cuda.synchronize()
                outer.barrier.wait()

            def allgather(self, buf, n):
                import torch
                torch.cuda.synchronize()
                outer.slots[r] = buf
                outer.barrier.wait()
                for q in range(outer.nranks):
                    if q != r:
                        buf[q * n:(q + 1) * n].copy_(outer.slots[q][q * n:(q + 1) * n])
                torch.cuda.synchronize()
                outer.barrier.wait()

        return _Rank(r, self.nranks, self.device)


# ---------------------------------------------------------------------------
# primitives and parity hooks

def kernel_block_apply(kernel: KernelSpec, targets, sources, shift, density, out, skip_coincident=False,
                       context: Optional[Context] = None):
    """kernel_block_apply (src/kernel.cpp:80-129) on the device; accumulates into `out`."""
    ctx = context or default_context()
    t = np.ascontiguousarray(targets, dtype=np.float64).reshape(-1, 3)
    s = np.ascontiguousarray(sources, dtype=np.float64).reshape(-1, 3)
    d = np.ascontiguousarray(density, dtype=np.float64).reshape(-1)
    sh = np.ascontiguousarray(shift, dtype=np.float64).reshape(3)
    o = np.ascontiguousarray(out, dtype=np.float64)
    err = _errbuf()
    _check(lib().pkgpu_kernel_block_apply(ctx._h, int(kernel.type), _ptr(t), len(t), _ptr(s), len(s), _ptr(sh),
                                          _ptr(d), _ptr(o), 1 if skip_coincident else 0, err, 1024), err)
    if o is not out:
        out[...] = o
    return out


def i8_moduli():
    """The pairwise-coprime moduli of the int8 M2L residue arithmetic."""
    out = (ctypes.c_int32 * 32)()
    n = lib().pkgpu_i8_moduli(out, 32)
    return [int(out[i]) for i in range(n)]


def i8_gather_gemm(A, B, rows_per_mod, zero_row, src, box0, R, context: Optional[Context] = None):
    """The int8 tensor-pipe gather-GEMM (test hook; device tensors with .data_ptr()):
    R[t][c][r] += sum_s sum_k A[t][s][r][k] B[t][row(s, c)][k] as balanced residues mod
    m_t, row = src[s][c] - box0 (zero_row when src < 0). A int8 [nmod][nmat][Ki][Ki],
    B int8 [nmod][rows_per_mod][Ki], src int32 [nslots][ncols], R int32 [nmod][ncols][Ki]."""
    ctx = context or default_context()
    nmod, nmat, Ki = A.shape[0], A.shape[1], A.shape[2]
    assert tuple(R.shape) == (nmod, src.shape[1], Ki)
    nslots, ncols = src.shape
    err = _errbuf()
    _check(lib().pkgpu_i8_gather_gemm(ctx._h, ctypes.c_void_p(A.data_ptr()), nmat, ctypes.c_void_p(B.data_ptr()),
                                      rows_per_mod, zero_row, Ki, nmod, ctypes.c_void_p(src.data_ptr()), ncols,
                                      box0, nslots, ncols, ctypes.c_void_p(R.data_ptr()), err, 1024), err)
    return R


def surface_points(p, center, edge):
    """surface_points (src/geometry.cpp:60-71), bit-exact."""
    c = np.ascontiguousarray(center, dtype=np.float64)
    out = np.empty((surface_point_count(p), 3))
    if lib().pkgpu_surface_points(p, _ptr(c), float(edge), _ptr(out)) != 0:
        raise ValueError("surface grid requires p >= 2")
    return out


def set_kifmm_factors(kernel: KernelSpec, p, up, dn, context: Optional[Context] = None):
    """Parity mode: inject (u, sigma, vt) factors of a_up and a_dn (SvdFactors layout)."""
    ctx = context or default_context()
    arrs = [np.ascontiguousarray(x, dtype=np.float64) for x in (*up, *dn)]
    err = _errbuf()
    _check(lib().pkgpu_set_kifmm_factors(ctx._h, int(kernel.type), p, *[_ptr(a) for a in arrs], err, 1024), err)


def get_kifmm_factors(kernel: KernelSpec, p, context: Optional[Context] = None):
    ctx = context or default_context()
    K = kernel.ks * surface_point_count(p)
    bufs = [np.empty((K, K)), np.empty(K), np.empty((K, K)), np.empty((K, K)), np.empty(K), np.empty((K, K))]
    err = _errbuf()
    _check(lib().pkgpu_get_kifmm_factors(ctx._h, int(kernel.type), p, *[_ptr(b) for b in bufs], err, 1024), err)
    return tuple(bufs[:3]), tuple(bufs[3:])


def kifmm_matrix(kernel: KernelSpec, p, which, i0=0, i1=0, i2=0, context: Optional[Context] = None):
    """Dense translation matrices for parity checks: which = a_up|a_dn|m2m|l2l|m2l|img."""
    ctx = context or default_context()
    code = {"a_up": 0, "a_dn": 1, "m2m": 2, "l2l": 3, "m2l": 4, "img": 5}[which]
    K = kernel.ks * surface_point_count(p)
    out = np.empty((K, K))
    err = _errbuf()
    _check(lib().pkgpu_kifmm_matrix(ctx._h, int(kernel.type), p, code, i0, i1, i2, _ptr(out), err, 1024), err)
    return out


def generate(kind, n, ks, seed=12345, nclusters=8, sigma=0.04, periodic_axes=(True, True, True)):
    """Seeded synthetic workload (SURVEY §8d protocol): kind = uniform|clusters|mixed."""
    kinds = {"uniform": 0, "clusters": 1, "mixed": 2}
    pts = np.empty((n, 3))
    q = np.empty(n * ks)
    ax = (ctypes.c_int * 3)(*[1 if a else 0 for a in periodic_axes])
    if lib().pkgpu_generate(kinds[kind], n, nclusters, sigma, ax, ks, seed, _ptr(pts), _ptr(q)) != 0:
        raise ValueError("generate: bad arguments")
    return pts, q


class FmmTree:
    """Device octree (FmmTree, include/pkifmm/fmm.hpp:31-101) with debug exports:
    structure_hash, BFS box table, leaf point lists and U/V/W/X lists."""

    def __init__(self, sources, targets, leaf_capacity=1000, context: Optional[Context] = None):
        self.ctx = context or default_context()
        s = np.ascontiguousarray(sources, dtype=np.float64).reshape(-1, 3)
        t = np.ascontiguousarray(targets, dtype=np.float64).reshape(-1, 3)
        h, err = ctypes.c_void_p(), _errbuf()
        _check(lib().pkgpu_tree_build(self.ctx._h, _ptr(s), len(s), _ptr(t), len(t), leaf_capacity, ctypes.byref(h),
                                      err, 1024), err)
        self._h = h
        self.n_sources, self.n_targets = len(s), len(t)

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value and _lib is not None:
            _lib.pkgpu_tree_free(self._h)

    def _info(self, want_hash=False):
        nb, nl, d, hsh = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int(), ctypes.c_uint64()
        lib().pkgpu_tree_info(self._h, ctypes.byref(nb), ctypes.byref(nl), ctypes.byref(d),
                              ctypes.byref(hsh) if want_hash else None)
        return nb.value, nl.value, d.value, hsh.value

    def box_count(self):
        return self._info()[0]

    def leaf_count(self):
        return self._info()[1]

    def depth(self):
        return self._info()[2]

    def structure_hash(self):
        return self._info(True)[3]

    def boxes(self):
        nb = self.box_count()
        table = np.empty((nb, 18), dtype=np.int32)
        s = np.empty(self.n_sources, dtype=np.int32)
        t = np.empty(self.n_targets, dtype=np.int32)
        lib().pkgpu_tree_boxes(self._h, _ptr(table), _ptr(s), _ptr(t))
        return table, s, t

    def lists(self, setup: Optional[PeriodicSetup], which):
        nb = self.box_count()
        off = np.empty(nb + 1, dtype=np.int64)
        st = setup._c() if setup is not None else None
        err = _errbuf()
        _check(lib().pkgpu_tree_lists(self._h, ctypes.byref(st) if st is not None else None, ord(which), _ptr(off),
                                      None, err, 1024), err)
        ent = np.empty((int(off[-1]), 4), dtype=np.int32)
        _check(lib().pkgpu_tree_lists(self._h, ctypes.byref(st) if st is not None else None, ord(which), _ptr(off),
                                      _ptr(ent), err, 1024), err)
        return off, ent
