set -u
OUT=gpurun_out/${TAG:-r02m}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for mode in "--streams 3" "--streams 2" "--batch 3" "--batch 2" "--streams 4 --reserve-sms 4"; do
  timeout 900 python bench.py --steps 9 --warmup 3 --no-cpu-baseline --no-dense $mode > $OUT/b.json 2> $OUT/b.err
  echo "mode=$mode rc=$?"
  OUT=$OUT python - <<'PY'
import json,os
d=json.loads(open(os.environ['OUT']+'/b.json').read().strip().splitlines()[-1])
print('  value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'single', round(d['single_stream']['value'],1), 'rho', d.get('final_rel_residual'))
PY
done
