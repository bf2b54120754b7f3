# Round-2: ncu --set full of the netscale step's big kernels (one launch each), after the same
# bench command exits 0 without ncu.  Read back with scripts/summarize_ncu_r2.py.
set -u
OUT=gpurun_out/${1:-nf}
mkdir -p $OUT
C="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --bulk-updates 0 --profile-steps 0"
$C > $OUT/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"${2:-tc_grad2p_kernel|tc_stats_kernel}" \
    --launch-skip ${3:-0} -c ${4:-2} -o $OUT/full $C > $OUT/ncu.log 2>&1
echo ncu_rc=$?
