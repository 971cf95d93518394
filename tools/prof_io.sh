cp abtest/libfeod_prof.so paper_2506_00746_b200/libfeod.so
REPS=${REPS:-1} ONLY=${ONLY:-} timeout 120 python tools/exp_variants.py ${WLD:-C3} > /tmp/pio.log 2>&1
grep "IO blk" /tmp/pio.log | tail -6
grep "CW mode 1" /tmp/pio.log | tail -8
grep "label" /tmp/pio.log
