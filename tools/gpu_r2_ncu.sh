# ncu evidence for the round-2 kernels (each run only after the same command exited 0 without ncu)
python tools/ens_rate.py 1024 4 > gpurun_out/plain1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"cluster_pair|fk_smem|torque_step" -s 6 -c 3 \
      -o gpurun_out/r2_c5_kernels python tools/ens_rate.py 1024 4 > gpurun_out/ncu1.log 2>&1
WATER=1 python tools/ens_rate.py 1024 2 > gpurun_out/plain2.log 2>&1 && \
  WATER=1 ncu --set full --clock-control none --import-source on -k regex:"bin_fused|solv_group" -s 2 -c 2 \
      -o gpurun_out/r2_c5w_kernels python tools/ens_rate.py 1024 2 > gpurun_out/ncu2.log 2>&1
python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/plain3.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_bench_launches.csv \
      python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/ncu3.log 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/r2_bench_launches.csv
