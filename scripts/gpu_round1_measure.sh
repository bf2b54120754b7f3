# Round-1 measurement pass: default bench line, per-workload lines, launch list, ncu captures.
set -u
mkdir -p gpurun_out/r1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r1/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r1/smoke.log 2>&1
python bench.py > gpurun_out/r1/bench_default.json 2> gpurun_out/r1/bench_default.err
for w in reacher humanoid sweep512 sweep1024 sweep2048 sweep4096 sweep8192 sweep16384 netscale; do
  timeout 300 python bench.py --workload $w --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/r1/bench_$w.json 2>/dev/null
done
for e in dot cos; do
  timeout 300 python bench.py --workload sweep16384 --energy $e --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/r1/bench_sweep16384_$e.json 2>/dev/null
  timeout 300 python bench.py --workload sweep4096 --energy $e --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/r1/bench_sweep4096_$e.json 2>/dev/null
done
timeout 300 python bench.py --workload sweep4096 --precision fp32 --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/r1/bench_sweep4096_fp32.json 2>/dev/null
timeout 300 python bench.py --workload ant --precision fp32 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/r1/bench_ant_fp32.json 2>/dev/null
# launch list (ncu, serialised, warm caches) of one ant step, then full captures of the top kernels
C="python bench.py --workload ant --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --profile-steps 0"
$C > gpurun_out/r1/plain_ant.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 50 -c 12 --csv --log-file gpurun_out/r1/launches_ant.csv $C > /dev/null 2>&1
$C > gpurun_out/r1/plain_ant2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'tc_cchain_kernel|tc_gradf_kernel|tc_stats_kernel|tc_dwg_kernel' -s 8 -c 5 -o gpurun_out/r1/ant_full $C > /dev/null 2>&1
C2="python bench.py --workload sweep16384 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --profile-steps 0"
$C2 > gpurun_out/r1/plain_16k.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 11 --csv --log-file gpurun_out/r1/launches_sweep16384.csv $C2 > /dev/null 2>&1
$C2 > gpurun_out/r1/plain_16k2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'tc_gradf_kernel|tc_stats_kernel|tc_chain_kernel|tc_dwg_kernel' -s 5 -c 5 -o gpurun_out/r1/sweep16384_full $C2 > /dev/null 2>&1
ls -la gpurun_out/r1
