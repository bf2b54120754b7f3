# two-call logits split count chosen for half the SMs (both sides share one launch / the GPU)
set -x
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q -k "bf16 or ticket" 2>&1 | tail -3
timeout 300 python bench.py --workload sweep16384 --energy dot --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1
timeout 300 python bench.py --workload sweep4096 --energy dot --steps 100 --warmup 10 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1
timeout 300 python bench.py --workload sweep8192 --energy dot --steps 50 --warmup 10 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1
timeout 300 python bench.py --workload netscale --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1
timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1
