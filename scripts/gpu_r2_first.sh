# Round-2 first pass: GPU tests, the default (netscale) bench line, the MUFU calibration.
set -u
mkdir -p gpurun_out/r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a/gpu.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mufu_bench scratch/mufu_bench.cu && /tmp/mufu_bench > gpurun_out/r2a/mufu_bench.txt 2>&1
timeout 300 python bench.py --steps 50 --warmup 5 --cpu-seconds 8 > gpurun_out/r2a/bench_netscale.json 2> gpurun_out/r2a/bench_netscale.err
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r2a/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2a/pytest_gpu.log
tail -5 gpurun_out/r2a/pytest_gpu.log
