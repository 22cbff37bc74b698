#!/bin/bash
# Per-kernel CUDA-event times of one Large solve (tools/quick_bench.py profile) for the default build
# and each experimental variant paper_2008_10275_b200/liblrcheb_<name>.so named on the command line.
cd "$(dirname "$0")/.."
for v in default "$@"; do
  if [ "$v" = default ]; then lib=""; else lib="$PWD/paper_2008_10275_b200/liblrcheb_$v.so"; fi
  echo "== $v"
  LRCHEB_LIB=$lib timeout 300 python tools/quick_bench.py profile large 2>&1 | grep -E "warm=True\]|ts_gram|ts_store|spmm " | head -5
done
