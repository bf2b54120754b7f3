# Adam: p / m / v of the first grid-stride element requested before the PDL wait
set -x
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for i in 1 2; do timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1; done
timeout 300 python bench.py --workload reacher --steps 300 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1
timeout 300 python bench.py --workload sweep4096 --steps 100 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1
timeout 300 python bench.py --precision fp32 --steps 100 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1
