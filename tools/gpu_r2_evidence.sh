# round-2 evidence refresh: bench line, ncu --set full of the C5 kernels, the bench launch list
python bench.py > gpurun_out/bench_r2c.log 2>&1; tail -c 600 gpurun_out/bench_r2c.log
python tools/ens_rate.py 1024 4 > gpurun_out/plain1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"cluster_pair|fk_smem|torque_step" -s 6 -c 3 \
      -o gpurun_out/r2c_c5_kernels python tools/ens_rate.py 1024 4 > gpurun_out/ncu1.log 2>&1
python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/plain3.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c_bench_launches.csv \
      python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/ncu3.log 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/*.csv
