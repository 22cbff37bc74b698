set -u
OUT=gpurun_out/${TAG:-r02e}; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1; echo build=$?
timeout 600 python tools/quick_bench.py large 20 > $OUT/plain.log 2>&1 && \
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:spmm_tma_kernel -s 2 -c 1 \
  -o $OUT/spmm_full -f python tools/quick_bench.py large 20 > $OUT/ncu_spmm.log 2>&1; echo ncu_spmm=$?
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:ts_kernel -s 45 -c 3 \
  -o $OUT/ts_full -f python tools/quick_bench.py large 20 > $OUT/ncu_ts.log 2>&1; echo ncu_ts=$?
ls -la $OUT
