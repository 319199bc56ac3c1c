timeout 120 ./tools/i8_peak > gpurun_out/r37_i8peak.jsonl 2>&1; cat gpurun_out/r37_i8peak.jsonl
