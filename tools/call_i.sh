set -u
OUT=gpurun_out/${TAG:-r02i}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo pytest=$?; tail -15 $OUT/pytest.log
timeout 300 python tools/k1_time.py large > $OUT/k1.log 2>&1; cat $OUT/k1.log
timeout 600 python tools/quick_bench.py profile large > $OUT/prof.log 2>&1; head -8 $OUT/prof.log
