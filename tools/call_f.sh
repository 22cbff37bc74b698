set -u
OUT=gpurun_out/${TAG:-r02f}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "apply or solve_small or solve_tiny" > $OUT/pytest.log 2>&1; echo pytest=$?; tail -2 $OUT/pytest.log
timeout 600 python tools/quick_bench.py large 20 > $OUT/qb.log 2>&1; echo qb=$?; grep K1 $OUT/qb.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo bench=$?; tail -c 300 $OUT/bench.err
OUT=$OUT python - <<'PY'
import json,os
d=json.loads(open(os.environ.get('OUT','gpurun_out/r02f')+'/bench.json').read().strip().splitlines()[-1])
print('value', d['value'], 'e2e', d['e2e']['value'], 'single', d['single_stream']['value'])
print({k: round(v['avg_ms'],3) for k,v in d['roofline_kernels'].items()})
PY
