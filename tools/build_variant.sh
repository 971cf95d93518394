#!/bin/bash
# Build libfeod with extra nvcc flags into abtest/libfeod_<name>.so (own object
# directory; the default build is untouched). Run it with FEOD_LIB=abtest/libfeod_<name>.so.
# usage: tools/build_variant.sh NAME -DFLAG=1 ...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
python -c "import sys; sys.path.insert(0,'.'); from paper_2506_00746_b200.build import build; build(extra=sys.argv[2:], lib=sys.argv[1])" "abtest/libfeod_$name.so" "$@"
