set -u
OUT=gpurun_out/${TAG:-r02l}; mkdir -p $OUT
L=$PWD/paper_2008_10275_b200
LRCHEB_LIB=$L/liblrcheb_wd.so timeout 180 python tools/solve_probe.py medium 4 > $OUT/probe.log 2>&1; echo wd=$?; head -c 600 $OUT/probe.log
timeout 120 python tools/solve_probe.py medium 10 >> $OUT/probe.log 2>&1; echo def=$?; tail -1 $OUT/probe.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo pytest=$?; tail -15 $OUT/pytest.log
timeout 300 python tools/k1_time.py large > $OUT/k1.log 2>&1; cat $OUT/k1.log
timeout 600 python tools/quick_bench.py profile large > $OUT/prof.log 2>&1; head -8 $OUT/prof.log
