# ncu --set full of split-K (weight-gradient) tc_gemm launches of the recurrent update
mkdir -p gpurun_out
TAG=${1:-r03e}
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:'kernel<\(int\)32' -s 0 -c ${GCNT:-3} -o gpurun_out/prof_${TAG}_gemmsk -f \
  python bench.py --workload ppo_rnn --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/prof_${TAG}_gemmsk.log 2>&1
echo "prof rc=$?"
