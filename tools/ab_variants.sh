#!/bin/bash
# A/B timing of experimental library variants (tools/build_variant.sh) on the Large config:
# K1 S2STEP launch time and the graph-captured solve's ms/iteration (tools/quick_bench.py).
# Usage (under gpurun): bash tools/ab_variants.sh TAG name1 name2 ...   ("default" = liblrcheb.so)
cd "$(dirname "$0")/.."
TAG=$1; shift
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
for v in "$@"; do
  if [ "$v" = default ]; then lib=""; else lib="$PWD/paper_2008_10275_b200/liblrcheb_$v.so"; fi
  echo "== $v" | tee -a "$OUT/ab.log"
  LRCHEB_LIB=$lib timeout 600 python tools/quick_bench.py large 20 2>&1 | grep -E "K1|solve N|Error|error" | tee -a "$OUT/ab.log"
done
