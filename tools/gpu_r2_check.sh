# full GPU test suite + smoke + the default bench line
python -m pytest tests -m gpu -q -rf > gpurun_out/gpu_tests.log 2>&1; tail -5 gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
python bench.py > gpurun_out/bench.log 2>&1; tail -c 3000 gpurun_out/bench.log
