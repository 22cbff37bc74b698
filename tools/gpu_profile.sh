#!/bin/bash
# One GPU round trip: the GPU test suite, the contract bench, the ncu launch list of the same bench
# command and one `--set full` capture each of the SpMM and the tall-skinny kernels.
# Usage (from the repo root, under gpurun):  bash tools/gpu_profile.sh TAG [skip-tests]
set -u
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
NCU=/usr/local/cuda/bin/ncu
if [ "${2:-}" != "skip-tests" ]; then
  timeout 2400 python -m pytest tests -m gpu -x -q --durations=0 > "$OUT/pytest_gpu.log" 2>&1
  echo "pytest_exit=$?"; tail -2 "$OUT/pytest_gpu.log"
fi
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
rc=$?
echo "bench_exit=$rc"; cat "$OUT/bench.json"
[ $rc -eq 0 ] || exit $rc
# launch list of the bench command (one stream: ncu serialises kernels anyway, and its injection
# crashed with three solver threads capturing graphs concurrently)
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
  --log-file "$OUT/launches.csv" python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-dense --streams 1 \
  > "$OUT/ncu_launches.log" 2>&1
echo "ncu_launches_exit=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:spmm_tma_kernel -s 3 -c 1 \
  -o "$OUT/spmm_full" -f python tools/quick_bench.py large 4 > "$OUT/ncu_spmm.log" 2>&1
echo "ncu_spmm_exit=$?"
# steady state (rank = cap): the 46th..48th tall-skinny launches of the first N = 20 solve
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:ts_kernel -s 45 -c 3 \
  -o "$OUT/ts_full" -f python tools/quick_bench.py large 20 > "$OUT/ncu_ts.log" 2>&1
echo "ncu_ts_exit=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:spmm_dense_kernel -c 1 \
  -o "$OUT/dense_full" -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --streams 1 > "$OUT/ncu_dense.log" 2>&1
echo "ncu_dense_exit=$?"
for r in spmm_full ts_full dense_full; do
  [ -f "$OUT/$r.ncu-rep" ] && $NCU -i "$OUT/$r.ncu-rep" --page raw --csv > "$OUT/${r}_raw.csv" 2>/dev/null
done
ls -la "$OUT"
