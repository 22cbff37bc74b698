#!/bin/bash
# Whole-job iterations/s of bench.py under different subset schedules (Large): independent concurrent
# streams vs f1 lockstep groups (batched SpMM), one or several groups at once.
cd "$(dirname "$0")/.."
for opts in "--streams 3" "--batch 3 --groups 2" "--batch 2 --groups 2" "--batch 2 --groups 3" "--batch 4 --groups 2"; do
  line=$(timeout 600 python bench.py --steps 12 --warmup 6 --no-cpu-baseline --no-dense $opts 2>/dev/null | tail -1)
  python3 -c "import json,sys; d=json.loads(sys.argv[2]); print(sys.argv[1], '->', round(d['value'],1), 'it/s, e2e', round(d['e2e']['value'],1))" "$opts" "$line" || echo "$opts failed"
done
