// Runs the reference's own experiment harness (src/experiments.cpp, unmodified) with
// pkifmm::evaluate resolved to the GPU shim. Usage:
//   pkifmm_dropin <experiment> [--p-list 8,10] [--out DIR] [--operator-dir DIR]
// Exit code follows tools/pkifmm.cpp cmd_experiment: 0 pass, 2 threshold failure, 1 error.
#include <cstdio>
#include <iostream>
#include <sstream>
#include <string>

#include "pkifmm/experiments.hpp"

int main(int argc, char **argv) {
    if (argc < 2) {
        std::cerr << "usage: pkifmm_dropin <experiment> [--p-list a,b] [--out DIR] [--operator-dir DIR]\n";
        return 1;
    }
    pkifmm::experiments::ExperimentOptions opt;
    opt.write_files = false;
    for (int i = 2; i + 1 < argc; i += 2) {
        const std::string k = argv[i], v = argv[i + 1];
        if (k == "--p-list") {
            std::stringstream ss(v);
            std::string tok;
            while (std::getline(ss, tok, ',')) opt.p_list.push_back(std::stoi(tok));
        } else if (k == "--out") {
            opt.out_dir = v;
            opt.write_files = true;
        } else if (k == "--operator-dir") {
            opt.operator_dir = v;
        } else if (k == "--threads") {
            opt.threads = std::stoi(v);
        }
    }
    try {
        const auto rep = pkifmm::experiments::run_experiment(argv[1], opt);
        for (const auto &c : rep.checks)
            std::printf("{\"experiment\": \"%s\", \"check\": \"%s\", \"pass\": %s, \"value\": %.17g, \"detail\": \"%s\"}\n",
                        rep.name.c_str(), c.name.c_str(), c.pass ? "true" : "false", c.value, c.detail.c_str());
        return rep.pass() ? 0 : 2;
    } catch (const std::exception &e) {
        std::printf("{\"experiment\": \"%s\", \"error\": \"%s\"}\n", argv[1], e.what());
        return 1;
    }
}
