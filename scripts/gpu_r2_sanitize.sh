# Round-2: compute-sanitizer, ONE tool per gpurun call (see B200_PROFILING.md), small shapes:
# the smoke() hot path (Reacher, cluster chains, fused stats / gradient at D = 64) and one
# D = 256 critic step (CTA-pair GEMM, tc_stats, tc_grad2, merge, grouped dW, Adam).
#   bash scripts/gpu_r2_sanitize.sh OUT TOOL
set -u
OUT=gpurun_out/${1:-san}
TOOL=${2:-memcheck}
mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 900 compute-sanitizer --tool $TOOL --target-processes all --print-limit 50 \
  python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/${TOOL}_smoke.log 2>&1
echo "smoke rc=$?" >> $OUT/${TOOL}_smoke.log
timeout 1200 compute-sanitizer --tool $TOOL --target-processes all --print-limit 50 \
  python -m pytest tests/test_gpu_parity.py -q -x -k "test_critic_step_bf16_grad2_d256 and l2-None and 1100" \
  > $OUT/${TOOL}_d256.log 2>&1
echo "d256 rc=$?" >> $OUT/${TOOL}_d256.log
tail -4 $OUT/${TOOL}_smoke.log $OUT/${TOOL}_d256.log
