# Round-2: one ncu --set full capture each of the netscale step's big kernels (after the same
# bench command exits 0 without ncu)
set -u
OUT=gpurun_out/${1:-ncu3}
mkdir -p $OUT
C="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --bulk-updates 0"
$C > $OUT/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${2:-tc_pgemm_kernel|tc_stats_kernel|tc_dwg_kernel}" -c ${3:-3} -o $OUT/full $C > $OUT/ncu.log 2>&1
echo ncu_rc=$?
