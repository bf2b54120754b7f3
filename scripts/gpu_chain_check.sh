set -x
python -m pytest tests -m gpu -x -q -k "bf16" 2>&1 | tail -15
for w in ant sweep4096 sweep16384; do
  timeout 300 python bench.py --workload $w --steps 300 --warmup 20 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-400
  CRL_NO_CHAIN=1 timeout 300 python bench.py --workload $w --steps 300 --warmup 20 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-400
done
