#!/bin/bash
# Headline sensitivity to the concurrent-subset schedule: streams x reserved SMs (Large, bench.py).
cd "$(dirname "$0")/.."
for st in 2 3 4; do
  for rs in 2 3 5; do
    line=$(timeout 600 python bench.py --steps 12 --warmup 6 --no-cpu-baseline --no-dense --streams $st --reserve-sms $rs 2>/dev/null | tail -1)
    python3 -c "import json,sys; d=json.loads(sys.argv[1]); print('streams', sys.argv[2], 'reserve', sys.argv[3], '->', round(d['value'],1), 'it/s')" "$line" $st $rs || echo "streams $st reserve $rs failed"
  done
done
