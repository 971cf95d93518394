#!/bin/bash
# In-kernel clock instrumentation of the plane kernel: build with tools/build_variant.sh prof -DFEOD_PROFILE_IO
FEOD_LIB=$PWD/abtest/libfeod_prof.so REPS=${REPS:-1} ONLY=${ONLY:-} timeout 120 python tools/exp_variants.py ${WLD:-C3} > /tmp/pio.log 2>&1
grep "IO blk" /tmp/pio.log | tail -6
grep "CW mode 1" /tmp/pio.log | tail -8
grep "label" /tmp/pio.log
