set -u
OUT=gpurun_out/r02a; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1; echo build=$?
timeout 1800 python -m pytest tests -m gpu -x -q -k "not vs_golden and not bench_configuration" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo pytest=$?; tail -4 $OUT/pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo bench=$?; tail -c 600 $OUT/bench.err
