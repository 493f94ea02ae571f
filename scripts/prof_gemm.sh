# ncu --set full of one tc_gemm launch of the recurrent collector (M = 49152 rows, N = 384)
mkdir -p gpurun_out
TAG=${1:-r02o}
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:gemm_ws_kernel -s ${GSKIP:-40} -c ${GCNT:-1} \
  -o gpurun_out/prof_${TAG}_gemm -f python bench.py --workload ppo_rnn --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/prof_${TAG}_gemm.log 2>&1
echo "prof rc=$?"
