set -u
OUT=gpurun_out/abl
mkdir -p $OUT
for d in 0 8 0 8; do
  CRL_G2P_DBG=$d python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/b$d.json 2>/dev/null
  python -c "import json; d=json.load(open('$OUT/b$d.json')); print('$d', d['value'], d['roofline']['stages_us'].get('grad_pair'), d['clocks']['sm_mhz'])"
done
CRL_NO_G2_WSYM=1 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/boff.json 2>/dev/null
python -c "import json; d=json.load(open('$OUT/boff.json')); print('off', d['value'], d['roofline']['stages_us'].get('grad_pair'), d['clocks']['sm_mhz'])"
