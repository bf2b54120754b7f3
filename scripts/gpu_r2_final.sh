# Round-2 final measurement pass: the whole GPU suite, the default (netscale) bench line with
# the oracle cpu_baseline, the other configurations, the netscale launch list and one
# `ncu --set full` capture of each top kernel (each after its command exited 0 without ncu).
set -u
OUT=gpurun_out/${1:-final}
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench_netscale.json 2> $OUT/bench_netscale.err; echo "bench rc=$?"
bash scripts/gpu_r2_configs.sh ${1:-final}/cfg > $OUT/cfg.txt 2>&1
bash scripts/gpu_r2_launches.sh ${1:-final}/ln > $OUT/launches.txt 2>&1
for k in tc_grad2p_kernel tc_stats_kernel; do
  bash scripts/gpu_r2_ncufull.sh ${1:-final}/ncu_$k "$k" 0 1 > /dev/null 2>&1
done
# tc_pdw_kernel runs twice per step: the stored-W column GEMM (first) and the dW / db launch
bash scripts/gpu_r2_ncufull.sh ${1:-final}/ncu_tc_pdw_gemm "tc_pdw_kernel" 0 1 > /dev/null 2>&1
bash scripts/gpu_r2_ncufull.sh ${1:-final}/ncu_tc_pdw_kernel "tc_pdw_kernel" 1 1 > /dev/null 2>&1
bash scripts/gpu_r2_ncufull.sh ${1:-final}/ncu_pg "tc_pgemm_kernel" 1 2 > /dev/null 2>&1
ls $OUT
