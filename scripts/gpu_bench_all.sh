# bench.py lines for every workload (default settings), into gpurun_out/r1b/
set -u
mkdir -p gpurun_out/r1b
for w in reacher humanoid sweep512 sweep1024 sweep2048 sweep4096 sweep8192 sweep16384 netscale; do
  timeout 300 python bench.py --workload $w --steps 300 --warmup 20 --no-cpu-baseline > gpurun_out/r1b/bench_$w.json 2>/dev/null
done
ls gpurun_out/r1b
