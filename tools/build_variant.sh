#!/bin/bash
# Build libfeod with extra nvcc flags into abtest/libfeod_<name>.so, then restore the default build.
# usage: tools/build_variant.sh NAME -DFLAG=1 ...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p abtest
touch paper_2506_00746_b200/csrc/plane_kernel.cuh
python -c "import sys; sys.path.insert(0,'.'); from paper_2506_00746_b200.build import build; build(extra=sys.argv[1:])" "$@"
cp paper_2506_00746_b200/libfeod.so abtest/libfeod_$name.so
