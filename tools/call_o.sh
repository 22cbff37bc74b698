set -u
OUT=gpurun_out/${TAG:-r02o}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1; echo build=$?
timeout 1200 python -m pytest tests/test_gpu_gmres.py tests/test_gpu_terms.py tests/test_gpu_batch.py -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo pytest=$?; tail -30 $OUT/pytest.log
