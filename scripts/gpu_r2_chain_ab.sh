# A/B: fused MLP chains vs per-layer (CTA-pair) GEMMs at the sweep batch sizes.
set -u
OUT=gpurun_out/${1:-chain}
mkdir -p $OUT
for wl in sweep16384 sweep4096; do
  for v in chain layer chain layer; do
    if [ $v = layer ]; then export CRL_NO_CHAIN=1; else unset CRL_NO_CHAIN; fi
    timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --bulk-updates 0 --workload $wl > $OUT/${wl}_$v.json 2> $OUT/${wl}_$v.err
    python -c "
import json; d=json.load(open('$OUT/${wl}_$v.json')); r=d['roofline']['stages_us']
print('$wl $v', d['value'], d['clocks']['sm_mhz'], {k: v for k, v in r.items() if v > 8})"
  done
done
unset CRL_NO_CHAIN
