# one-launch two-sided statistics (tc_logits_lse_pair): parity + ant / dot benches
set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "bf16" 2>&1 | tail -5
timeout 300 python bench.py --steps 300 --warmup 10 2>/dev/null | tail -1
timeout 300 python bench.py --workload reacher --steps 300 --warmup 10 2>/dev/null | tail -1
timeout 300 python bench.py --workload sweep16384 --energy dot --steps 20 --warmup 5 2>/dev/null | tail -1
timeout 300 python bench.py --workload netscale --steps 10 --warmup 3 2>/dev/null | tail -1
