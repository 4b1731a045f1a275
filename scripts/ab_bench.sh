# same-box A/B of env toggles on the BERT bench line: value / e2e (ms) per run, alternating
# Usage: scripts/ab_bench.sh "ENV_A" "ENV_B" [rounds]
A=${1:-X=1}; B=${2:-X=1}; N=${3:-3}
for i in $(seq $N); do
  for cfg in "$A" "$B"; do
    env $cfg python bench.py --no-sweep --no-cpu-baseline --steps 10 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg', round(d['value']*1e3,3), round(d['e2e']['value']*1e3,3))"
  done
done
