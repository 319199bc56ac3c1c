R=${R:-r45}
ll() { timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:m2l_i8 --csv --log-file gpurun_out/${R}_$1.csv python tools/run_cfg2.py --evals 1 --warm 1 > /dev/null 2>&1; echo "$1 $(python tools/launch_times.py gpurun_out/${R}_$1.csv)"; }
ll base
PKGPU_I8_DEBUG=16 ll oneop
PKGPU_I8_DEBUG=1 ll nogather
PKGPU_I8_DEBUG=2 ll noop
PKGPU_I8_DEBUG=3 ll noloads
PKGPU_I8_DEBUG=4 ll noatomics
PKGPU_I8_PAIR=3 ll dual
PKGPU_I8_PAIR=3 PKGPU_I8_DEBUG=16 ll dual_oneop
PKGPU_I8_PAIR=2 ll mc
PKGPU_I8_PREFETCH=8 ll pf8
