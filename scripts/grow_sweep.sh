# grid-wave window sweep: growth factor after a clean full wave (TSAT_WIN_GROW) and first
# window (TSAT_WIN0) and largest window (TSAT_WIN_MAX); BERT bench line and the configs[4] search
for cfg in "16 4096 4194304" "16 16384 1048576" "16 8192 1048576" "16 16384 4194304" "16 4096 4194304" "16 16384 1048576" "16 8192 1048576" "16 16384 4194304"; do
  set -- $cfg
  echo "grow=$1 win0=$2 max=$3"
  TSAT_WIN_GROW=$1 TSAT_WIN0=$2 TSAT_WIN_MAX=$3 python bench.py --no-sweep --no-cpu-baseline --steps 8 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('  bert', round(d['value']*1e3,3), round(d['e2e']['value']*1e3,3))"
  TSAT_WIN_GROW=$1 TSAT_WIN0=$2 TSAT_WIN_MAX=$3 python bench.py --workload synth10m --no-sweep --no-cpu-baseline --steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('  10m', round(d['value']*1e3,3), round(d['e2e']['value']*1e3,3), d['kernel_groups_ms_per_step']['apply_wave'])"
done
