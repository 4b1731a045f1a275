# cycle-check peel variants on BERT: barrier-free shared-memory walk threads (TSAT_PEEL_THREADS) and the
# level-synchronous walk (TSAT_PEEL_SYNC); bench line value / e2e (ms)
for cfg in "X=1" "TSAT_PEEL_THREADS=512" "TSAT_PEEL_THREADS=256" "TSAT_PEEL_SYNC=1" "X=1" "TSAT_PEEL_THREADS=512" "TSAT_PEEL_THREADS=256" "TSAT_PEEL_SYNC=1"; do
  env $cfg python bench.py --no-sweep --no-cpu-baseline --steps 8 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg', round(d['value']*1e3,3), round(d['e2e']['value']*1e3,3), d['kernel_groups_ms_per_step']['cycles'])"
done
