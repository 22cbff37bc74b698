set -u
OUT=gpurun_out/${TAG:-r02n}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1; echo build=$?
timeout 1200 python -m pytest tests/test_gpu_terms.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo pytest=$?; tail -25 $OUT/pytest.log
timeout 600 python bench.py --config small4 --steps 6 --warmup 3 --no-dense > $OUT/b_small4.json 2> $OUT/b_small4.err; echo b4=$?; tail -c 400 $OUT/b_small4.err
timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-dense > $OUT/b_large.json 2> $OUT/b_large.err; echo bl=$?; tail -c 400 $OUT/b_large.err
for f in b_small4 b_large; do OUT=$OUT F=$f python - <<'PY'
import json,os
d=json.loads(open(os.environ['OUT']+'/'+os.environ['F']+'.json').read().strip().splitlines()[-1])
print(os.environ['F'], 'value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'single', round(d['single_stream']['value'],1), 'f1', d.get('f1_batched') and round(d['f1_batched']['value'],1), 'rho', d.get('final_rel_residual'))
print({k: round(v['avg_ms'],3) for k,v in d['roofline_kernels'].items()})
PY
done
