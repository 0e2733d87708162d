#!/bin/bash
# A/B timing of library builds on one box: tools/ab/lib_<name>.so copied over
# the in-tree library in turn, bench.py run for each (same box, same clocks).
#   bash tools/ab_run.sh WORKLOAD name1 name2 ...
W=$1; shift
cp paper_2604_07173_b200/liblora_server.so /tmp/lib_keep.so
for n in "$@"; do
  cp tools/ab/lib_$n.so paper_2604_07173_b200/liblora_server.so
  LORA_BINDING_LENIENT=1 timeout 120 python bench.py --workload $W --steps 50 --warmup 5 --no-cpu-baseline \
      --e2e-steps 0 > gpurun_out/ab_$n.json 2> gpurun_out/ab_$n.err
done
cp /tmp/lib_keep.so paper_2604_07173_b200/liblora_server.so
