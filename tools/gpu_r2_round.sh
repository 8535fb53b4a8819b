# full GPU test suite + the bench, then the kernel-choice sweep (old vs cluster) over batch sizes
python -m pytest tests -m gpu -q -rf -x > gpurun_out/gpu_tests_r2b.log 2>&1; tail -5 gpurun_out/gpu_tests_r2b.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2b.log 2>&1; tail -c 1500 gpurun_out/bench_r2b.log
for B in 128 192 256 384; do KFB200_CLUSTER=0 python tools/ens_rate.py $B 16; python tools/ens_rate.py $B 16; done
