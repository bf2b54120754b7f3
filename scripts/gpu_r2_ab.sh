# Alternating A/B of one knob on the default bench line (device value and e2e), N rounds.
set -u
VAR=$1; N=${2:-4}; OUT=gpurun_out/${3:-ab}
mkdir -p $OUT
for r in $(seq $N); do
  for v in on off; do
    if [ $v = off ]; then export $VAR=1; else unset $VAR; fi
    timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --bulk-updates 0 --profile-steps 0 > $OUT/b_$v.json 2>/dev/null
    python -c "
import json; d=json.load(open('$OUT/b_$v.json')); print('$v', d['value'], d['e2e']['value'], d['clocks']['sm_mhz'])"
  done
done
unset $VAR
