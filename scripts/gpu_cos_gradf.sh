set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "bf16" 2>&1 | tail -5
for e in l2 cos; do timeout 300 python bench.py --workload sweep16384 --energy $e --steps 20 --warmup 5 2>/dev/null | tail -1; done
for e in cos; do timeout 300 python bench.py --workload sweep4096 --energy $e --steps 50 --warmup 5 2>/dev/null | tail -1; timeout 300 python bench.py --energy $e --steps 200 --warmup 10 2>/dev/null | tail -1; done
