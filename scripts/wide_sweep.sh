# single-CTA loop -> grid path hand-over sweep (TSAT_WIDE_AFTER: clean full windows before the hand-over); BERT bench line
for wa in 8 2 4 16 8 2 4 16; do
  TSAT_WIDE_AFTER=$wa python bench.py --no-sweep --no-cpu-baseline --steps 8 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('wide_after=$wa bert', round(d['value']*1e3,3), round(d['e2e']['value']*1e3,3))"
done
