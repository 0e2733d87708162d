#!/bin/bash
# Regenerate the judged evidence under profiles/ on a B200 (run via gpurun):
#   bench lines (our arm, reference arm), ncu launch lists per workload,
#   ncu --set full summaries of the kernels of the default workload.
#   usage: bash tools/profile_round.sh TAG     (e.g. r1)
set -u
TAG=${1:-r1}
OUT=gpurun_out/prof
mkdir -p $OUT
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
for w in mixtral_sharded mixtral_decode mixtral_prefill llama_decode; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 \
      > $OUT/bench_$w.json 2> $OUT/bench_$w.err
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file $OUT/launches_$w.csv \
      python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
done
# one full capture per kernel kind of the default workload (after warm-up)
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'segment_kernel|simt_shrink|simt_expand|tc_shrink|tc_vreduce|tc_expand' -s 6 -c 6 \
    -o $OUT/full_mixtral_sharded python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 \
    > $OUT/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'simt_shrink|simt_expand|tc_shrink|tc_expand' -s 4 -c 4 \
    -o $OUT/full_mixtral_prefill python bench.py --workload mixtral_prefill --steps 2 --warmup 3 --no-cpu-baseline \
    --e2e-steps 0 > $OUT/ncu_full_prefill.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'simt_shrink|simt_expand' -s 4 -c 2 \
    -o $OUT/full_llama_decode python bench.py --workload llama_decode --steps 2 --warmup 3 --no-cpu-baseline \
    --e2e-steps 0 > $OUT/ncu_full_llama.log 2>&1
# summaries on the box; the .ncu-rep files stay there (gpurun_out/ is capped at 64 MiB)
for r in full_mixtral_sharded full_mixtral_prefill full_llama_decode; do
  [ -f $OUT/$r.ncu-rep ] && python tools/ncu_summary.py $OUT/$r.ncu-rep > $OUT/sum_$r.txt 2>&1
done
mkdir -p /tmp/ncu_reps && mv $OUT/*.ncu-rep /tmp/ncu_reps/ 2>/dev/null
echo done
