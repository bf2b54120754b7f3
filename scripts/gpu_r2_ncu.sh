# ncu captures of the netscale step's kernels (run only after the same command exits 0 without ncu)
set -u
OUT=gpurun_out/${1:-ncu}
REGEX=${2:-'tc_grad2|tc_stats'}
mkdir -p $OUT
C="python bench.py --steps 2 --warmup 1 --profile-steps 0 --no-e2e --no-cpu-baseline --bulk-updates 0 --sample-every 1"
$C > $OUT/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$REGEX" -c ${3:-2} -o $OUT/full $C > $OUT/ncu.log 2>&1
echo ncu_rc=$?
ls -la $OUT
