#!/bin/bash
# Build an experimental variant of liblrcheb.so with extra -D flags (selected at run time by the
# binding's LRCHEB_LIB): tools/build_variant.sh NAME -DFOO=1 ...
set -e
NAME=$1; shift
cd "$(dirname "$0")/.."
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -O3 --threads 0 "$@" -shared -o paper_2008_10275_b200/liblrcheb_$NAME.so paper_2008_10275_b200/csrc/*.cu
