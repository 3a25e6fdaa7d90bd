#!/bin/bash
# Run bench.py under several env settings; one JSON line per setting into
# gpurun_out/sweep.jsonl (tagged with the env string).  Usage:
#   scripts/bench_sweep.sh "ENV1=a ENV2=b" "ENV1=c" ...   (extra bench args in BENCH_ARGS)
mkdir -p gpurun_out
for cfg in "$@"; do
  line=$(env $cfg timeout 600 python bench.py --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline $BENCH_ARGS 2>gpurun_out/sweep_err.txt | tail -1)
  python - "$cfg" "$line" <<'PY' >> gpurun_out/sweep.jsonl
import json, sys
cfg, line = sys.argv[1], sys.argv[2]
try:
    d = json.loads(line)
    out = {"env": cfg, "value": d["value"], "ms": d["ms_per_step"], "gemm_frac": d["roofline"]["frac"],
           "rs_ms": d["kernels"]["rs_adam"]["ms_per_step"], "ops": d["kernels"]["op_ms_per_step"],
           "sm_mhz": d["clocks"]["sm_mhz"], "reasons": d["clocks"]["reasons"]}
except Exception as e:
    out = {"env": cfg, "error": str(e), "line": line[-300:]}
print(json.dumps(out))
PY
done
