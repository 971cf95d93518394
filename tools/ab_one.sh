bash tools/prof_io.sh | grep -E "IO blk" | head -6
cp abtest/libfeod_minb3.so paper_2506_00746_b200/libfeod.so
timeout 120 python tools/exp_variants.py C3 C2 | grep label
