#!/bin/bash
# Time the K1 S2STEP launch (tools/quick_bench.py, Large, r = 60) for the default build and every
# experimental variant paper_2008_10275_b200/liblrcheb_<name>.so given on the command line.
cd "$(dirname "$0")/.."
for v in default "$@"; do
  if [ "$v" = default ]; then lib=""; else lib="$PWD/paper_2008_10275_b200/liblrcheb_$v.so"; fi
  echo "== $v"
  LRCHEB_LIB=$lib timeout 300 python tools/quick_bench.py large 20 2>&1 | grep -E "K1|solve N|Error"
done
