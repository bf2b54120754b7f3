# step-graph edge experiments (memset node removed; no fork / join without second-stream work)
set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "bf16 or ticket" 2>&1 | tail -3
for i in 1 2; do timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1; done
timeout 300 python bench.py --workload reacher --steps 300 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1
timeout 300 python bench.py --workload sweep4096 --steps 100 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1
timeout 300 python bench.py --workload sweep16384 --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1
