mkdir -p gpurun_out
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:probe_kernel -s 5 -c 1 -o gpurun_out/prof_r02d_mpeprobe -f python bench.py --workload mpe --steps 1000 --warmup 5 --no-e2e --no-cpu > gpurun_out/prof_r02d.log 2>&1; echo rc=$?
