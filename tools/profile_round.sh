#!/bin/bash
# Regenerate the judged evidence under profiles/ on a B200 (run via gpurun):
#   the default bench line (our arm, with the secondary configs and E10/E13),
#   the reference arm, an ncu launch list per workload (+ DRAM bytes per
#   launch), ncu --set full summaries of the kernels of each workload.
#   usage: bash tools/profile_round.sh TAG     (e.g. r2)
set -u
TAG=${1:-r2}
OUT=gpurun_out/prof
mkdir -p $OUT
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench_default.json 2> $OUT/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
timeout 600 python bench.py --force-sharded --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --no-secondary \
    > $OUT/bench_push_loopback.json 2> $OUT/bench_push_loopback.err
for w in mixtral_sharded mixtral_decode mixtral_prefill llama_decode; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-secondary \
      > $OUT/bench_$w.json 2> $OUT/bench_$w.err
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file $OUT/launches_$w.csv \
      python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-secondary --no-graph \
      > /dev/null 2>&1
done
# one full capture per kernel kind of each workload (after warm-up)
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'segment_kernel|simt_shrink|simt_expand|tc_shrink|tc_vreduce|tc_expand' -s 6 -c 6 \
    -o /tmp/full_mixtral_sharded python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-secondary \
    --no-graph > $OUT/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'simt_shrink|simt_expand|tc_shrink|tc_expand' -s 4 -c 4 \
    -o /tmp/full_mixtral_prefill python bench.py --workload mixtral_prefill --steps 2 --warmup 3 --no-cpu-baseline \
    --e2e-steps 0 --no-secondary --no-graph > $OUT/ncu_full_prefill.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'simt_shrink|simt_expand|tc_shrink|tc_expand' -s 5 -c 4 \
    -o /tmp/full_mixtral_decode python bench.py --workload mixtral_decode --steps 2 --warmup 3 --no-cpu-baseline \
    --e2e-steps 0 --no-secondary --no-graph > $OUT/ncu_full_decode.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'simt_shrink|simt_expand' -s 4 -c 2 \
    -o /tmp/full_llama_decode python bench.py --workload llama_decode --steps 2 --warmup 3 --no-cpu-baseline \
    --e2e-steps 0 --no-secondary --no-graph > $OUT/ncu_full_llama.log 2>&1
# the tcgen05 chain at r = 128 (prefill shapes)
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'tc_shrink|tc_expand' -s 2 -c 2 \
    -o /tmp/full_prefill_r128 python tools/prefill_rank.py 128 > $OUT/ncu_full_r128.log 2>&1
timeout 600 python tools/prefill_rank.py > $OUT/prefill_rank.json 2> $OUT/prefill_rank.err
# summaries on the box; the .ncu-rep files stay in /tmp there (gpurun_out/ is capped at 64 MiB)
for r in full_mixtral_sharded full_mixtral_prefill full_mixtral_decode full_llama_decode full_prefill_r128; do
  [ -f /tmp/$r.ncu-rep ] && python tools/ncu_summary.py /tmp/$r.ncu-rep > $OUT/sum_$r.txt 2>&1
done
echo done
