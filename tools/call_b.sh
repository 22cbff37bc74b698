set -u
OUT=gpurun_out/${TAG:-r02d}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1; echo build=$?
./tools/microbench/dmma_layout > $OUT/layout.json 2>&1; echo layout=$?; cat $OUT/layout.json
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo pytest=$?; tail -4 $OUT/pytest.log
timeout 600 python tools/quick_bench.py large 20 > $OUT/qb.log 2>&1; echo qb=$?; cat $OUT/qb.log
timeout 600 python tools/quick_bench.py profile large > $OUT/prof.log 2>&1; echo prof=$?; cat $OUT/prof.log
