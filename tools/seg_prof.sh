python tools/seg_timing.py
cp paper_2604_07173_b200/liblora_server.so /tmp/keep.so
cp tools/ab/lib_segprof.so paper_2604_07173_b200/liblora_server.so
python tools/seg_timing.py 2>&1 | sort | uniq -c | sort -rn | head -30
cp /tmp/keep.so paper_2604_07173_b200/liblora_server.so
