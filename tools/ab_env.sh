#!/bin/bash
# A/B of run-time switches on one box: each variant is "name:VAR=val,VAR2=val" (or "name:" for none),
# every workload run twice per variant, interleaved.
#   bash tools/ab_env.sh "w1 w2" base: v1:LORA_EXPAND_V1=1
WS=$1; shift
mkdir -p gpurun_out/ab
for w in $WS; do
  for rep in 1 2; do
    for v in "$@"; do
      n=${v%%:*}; envs=${v#*:}
      f=gpurun_out/ab/${w}_${n}_$rep.json
      env ${envs//,/ } timeout 120 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline \
          --e2e-steps 0 --no-secondary > $f 2> ${f%.json}.err
      python - "$w" "$n" "$rep" $f <<'PY' >> gpurun_out/ab/summary.txt
import json, sys
w, n, rep, f = sys.argv[1:]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    k = " ".join(f"{a}={b['ms_per_launch']*1e3:.1f}us" for a, b in d.get("kernels", {}).items())
    print(f"{w:16s} {n:10s} {rep} ms/step {d['ms_per_step']:.4f}  {k}")
except Exception as e:
    print(w, n, rep, "ERR", e)
PY
    done
  done
done
cat gpurun_out/ab/summary.txt
