#!/bin/bash
# Copy the results of tools/profile_round.sh (gpurun_out/prof) into profiles/
# (only files that came back; nothing is overwritten with an empty file).
TAG=${1:-r2}
P=gpurun_out/prof
for w in mixtral_sharded mixtral_decode mixtral_prefill llama_decode; do
  [ -s $P/launches_$w.csv ] && python tools/launch_list.py $P/launches_$w.csv $w profiles/${TAG}_launches_$w.txt \
      --traffic profiles/ncu_traffic.json > /dev/null
  [ -s $P/bench_$w.json ] && tail -1 $P/bench_$w.json > profiles/${TAG}_bench_$w.json
done
[ -s $P/bench_default.json ] && tail -1 $P/bench_default.json > profiles/${TAG}_bench_default.json
[ -s $P/bench_reference.json ] && tail -1 $P/bench_reference.json > profiles/${TAG}_bench_reference.json
[ -s $P/sum_full_mixtral_sharded.txt ] && cp $P/sum_full_mixtral_sharded.txt profiles/${TAG}_ncu_summary_mixtral_sharded.txt
[ -s $P/sum_full_mixtral_decode.txt ] && cp $P/sum_full_mixtral_decode.txt profiles/${TAG}_ncu_summary_mixtral_decode.txt
[ -s $P/bench_push_loopback.json ] && tail -1 $P/bench_push_loopback.json > profiles/${TAG}_bench_push_loopback.json
[ -s $P/sum_full_mixtral_prefill.txt ] && cp $P/sum_full_mixtral_prefill.txt profiles/${TAG}_ncu_summary_mixtral_prefill.txt
[ -s $P/sum_full_llama_decode.txt ] && cp $P/sum_full_llama_decode.txt profiles/${TAG}_ncu_summary_llama_decode.txt
[ -s $P/sum_full_prefill_r128.txt ] && cp $P/sum_full_prefill_r128.txt profiles/${TAG}_ncu_summary_prefill_r128.txt
[ -s $P/prefill_rank.json ] && tail -1 $P/prefill_rank.json > profiles/${TAG}_prefill_rank_sweep.json
true
