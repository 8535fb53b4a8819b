# round-2 evidence refresh: GPU suite, bench line, ncu --set full of the C5 kernels (one
# whole-batch launch each: KFB200_BRANCHES=1, so the eager and graph launches are the
# bench's 1024-trajectory kernels), the bench launch list
python -m pytest tests -m gpu -q 2>&1 | tail -2
python bench.py > gpurun_out/bench_r2n.log 2>&1; tail -c 300 gpurun_out/bench_r2n.log
KFB200_BRANCHES=1 python tools/ens_rate.py 1024 4 > gpurun_out/plain1.log 2>&1 && \
  KFB200_BRANCHES=1 ncu --set full --clock-control none --import-source on -k regex:"cluster_pair|fk_smem|torque_step" -s 6 -c 3 \
      -o gpurun_out/r2n_c5_kernels python tools/ens_rate.py 1024 4 > gpurun_out/ncu1.log 2>&1
python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/plain3.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2n_bench_launches.csv \
      python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/ncu3.log 2>&1
ls -la gpurun_out/r2n*
bash tools/gpu_bsweep.sh > gpurun_out/bsweep_r2n.log 2>&1
TAG=r2n bash tools/gpu_ncu_solv.sh > gpurun_out/solv_r2n_plain.log 2>&1
