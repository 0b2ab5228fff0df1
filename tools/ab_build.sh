#!/bin/bash
# Build an A/B variant of the library from the same sources with extra nvcc flags:
#   tools/ab_build.sh NAME "-DFLAG=1 ..."   ->  ab/NAME/libapmg_cuda.so  (select with APMG_LIB=...)
set -e
cd "$(dirname "$0")/.."
NAME=$1; FLAGS=$2
make -s -j8 LIB=ab/$NAME/libapmg_cuda.so EXTRA="$FLAGS" BUILD=build_ab/$NAME ab/$NAME/libapmg_cuda.so
