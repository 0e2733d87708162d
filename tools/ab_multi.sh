#!/bin/bash
# A/B over several workloads, each variant twice (interleaved) to see the noise.
#   bash tools/ab_multi.sh "w1 w2" name1 name2 ...
WS=$1; shift
mkdir -p gpurun_out/ab
cp paper_2604_07173_b200/liblora_server.so /tmp/lib_keep.so
for w in $WS; do
  for rep in 1 2; do
    for n in "$@"; do
      cp tools/ab/lib_$n.so paper_2604_07173_b200/liblora_server.so
      LORA_BINDING_LENIENT=1 timeout 120 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline \
          --e2e-steps 0 --no-secondary > gpurun_out/ab/${w}_${n}_$rep.json 2> gpurun_out/ab/${w}_${n}_$rep.err
      python - "$w" "$n" "$rep" gpurun_out/ab/${w}_${n}_$rep.json <<'PY' >> gpurun_out/ab/summary.txt
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
cp /tmp/lib_keep.so paper_2604_07173_b200/liblora_server.so
cat gpurun_out/ab/summary.txt
