#!/bin/bash
# Round evidence on one B200: gpu tests, bench lines for every workload, launch lists and one
# `ncu --set full` capture per step kernel (SMAX captured in steady state, after 30 launches).
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_${TAG}.log 2>&1; tail -2 gpurun_out/pytest_gpu_${TAG}.log
: > gpurun_out/bench_${TAG}.jsonl
for w in smax3m mpe mpe_large overcooked smax2s3z smax27m ippo ippo_oc; do
  timeout 600 python bench.py --workload $w --steps 30 --warmup 5 2>/dev/null | grep '^{' >> gpurun_out/bench_${TAG}.jsonl
done
timeout 600 python bench.py --workload smax27m --n-envs 16384 --steps 10 --warmup 3 2>/dev/null | grep '^{' >> gpurun_out/bench_${TAG}.jsonl
timeout 600 python bench.py --workload mpe --per-step --steps 30 --warmup 5 --no-cpu 2>/dev/null | grep '^{' >> gpurun_out/bench_${TAG}.jsonl
timeout 600 python bench.py --workload ppo --steps 10 --warmup 3 2>/dev/null | grep '^{' >> gpurun_out/bench_${TAG}.jsonl
timeout 600 python bench.py --workload ppo_rnn --steps 3 --warmup 3 2>/dev/null | grep '^{' >> gpurun_out/bench_${TAG}.jsonl
timeout 600 python bench.py --workload ppo_smax --steps 10 --warmup 3 2>/dev/null | grep '^{' >> gpurun_out/bench_${TAG}.jsonl
timeout 600 python bench.py --workload ppo_oc --steps 5 --warmup 3 2>/dev/null | grep '^{' >> gpurun_out/bench_${TAG}.jsonl
timeout 300 python bench.py --impl reference --workload smax3m --steps 3 --warmup 1 2>/dev/null | grep '^{' >> gpurun_out/bench_${TAG}.jsonl
timeout 300 python bench.py --impl reference --workload ippo_oc --steps 1 --warmup 1 2>/dev/null | grep '^{' >> gpurun_out/bench_${TAG}.jsonl
timeout 300 python bench.py --impl reference --workload ppo --steps 2 --warmup 3 2>/dev/null | grep '^{' >> gpurun_out/bench_${TAG}.jsonl
timeout 300 python bench.py --impl reference --workload ppo_rnn --steps 1 --warmup 3 2>/dev/null | grep '^{' >> gpurun_out/bench_${TAG}.jsonl
timeout 300 python bench.py --impl reference --workload ppo_smax --steps 1 --warmup 3 2>/dev/null | grep '^{' >> gpurun_out/bench_${TAG}.jsonl
timeout 300 python bench.py --impl reference --workload ppo_oc --steps 1 --warmup 3 2>/dev/null | grep '^{' >> gpurun_out/bench_${TAG}.jsonl
timeout 600 python scripts/ippo_oc_time.py 4096 SMAX_27m_vs_30m > gpurun_out/ippo27m_${TAG}.txt 2>&1
wc -l gpurun_out/bench_${TAG}.jsonl
NCU=/usr/local/cuda/bin/ncu
for w in smax3m smax2s3z mpe_large overcooked smax27m; do
  SKIP=4; [[ $w == smax* ]] && SKIP=30
  timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/launches_${TAG}_$w.csv python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu \
    > /dev/null 2>&1
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:step_kernel -s $SKIP -c 1 \
    -o gpurun_out/prof_${TAG}_$w -f python bench.py --workload $w --steps 3 --warmup 30 --no-e2e --no-cpu \
    > /dev/null 2>&1
done
bash scripts/prof_ippo.sh ${TAG} > /dev/null 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_ppo.csv \
  python bench.py --workload ppo --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_ppo_smax.csv \
  python bench.py --workload ppo_smax --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:ppo_update_tc -s 20 -c 1 \
  -o gpurun_out/prof_${TAG}_ppo_smax_update -f python bench.py --workload ppo_smax --steps 1 --warmup 3 --no-cpu --no-e2e \
  > /dev/null 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:ppo_update_tc -s 20 -c 1 \
  -o gpurun_out/prof_${TAG}_ppo_update -f python bench.py --workload ppo --steps 1 --warmup 3 --no-cpu --no-e2e \
  > /dev/null 2>&1
# summarise the step-kernel captures here and keep only what fits gpurun's 64 MiB return
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:probe_kernel -s 5 -c 1 \
  -o gpurun_out/prof_${TAG}_mpeprobe -f python bench.py --workload mpe --steps 1000 --warmup 5 --no-e2e --no-cpu > /dev/null 2>&1
GSKIP=3000 bash scripts/prof_gemm.sh ${TAG} > /dev/null 2>&1
# the wide-input update: launch list of one Overcooked PPO step, full captures of its two layer-1 GEMMs
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv \
  --log-file gpurun_out/launches_${TAG}_ppo_oc.csv python scripts/ppo_oc_time.py 4096 > /dev/null 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemm_ws_kernel -s 0 -c 1 \
  -o gpurun_out/prof_${TAG}_gemm_z1 -f python scripts/gemm_shapes.py 262144 > /dev/null 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemm_ws_kernel -s 21 -c 1 \
  -o gpurun_out/prof_${TAG}_gemm_dw1 -f python scripts/gemm_shapes.py 262144 > /dev/null 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:policy_tc_wide -s 10 -c 1 \
  -o gpurun_out/prof_${TAG}_wide27m -f python scripts/ippo_oc_time.py 1024 SMAX_27m_vs_30m > /dev/null 2>&1
LTAG=${TAG} SKIP=5000 CNT=6000 bash scripts/rnn_launches.sh > /dev/null 2>&1
python scripts/ncu_summary.py ${TAG} smax3m smax2s3z mpe_large overcooked smax27m > /dev/null 2>&1
mkdir -p gpurun_out/summary_${TAG}
cp profiles/${TAG}_* profiles/ncu_traffic.json profiles/ncu_metrics.json gpurun_out/summary_${TAG}/ 2>/dev/null
# a markdown brief of every capture, then keep only three reports (gpurun returns <= 64 MiB)
for r in gpurun_out/prof_${TAG}_*.ncu-rep; do
  b=$(basename $r .ncu-rep); python scripts/ncu_brief.py $r ${b#prof_${TAG}_} > gpurun_out/summary_${TAG}/brief_${b}.md 2>&1
done
python scripts/ncu_srcsum.py gpurun_out/prof_${TAG}_smax3m.ncu-rep 65536 45 > gpurun_out/summary_${TAG}/srcsum_smax3m.txt 2>&1
for r in gpurun_out/prof_${TAG}_*.ncu-rep; do
  case $r in *_smax3m.ncu-rep|*_gemm_dw1.ncu-rep|*_wide27m.ncu-rep) ;; *) rm -f $r ;; esac
done
du -sh gpurun_out
ls gpurun_out | grep ${TAG}
