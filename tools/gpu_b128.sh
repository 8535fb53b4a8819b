# B=128 strong-scaling floor: rate, eager phase times, and a per-kernel launch list
python tools/ens_rate.py 128 16 > gpurun_out/b128.log 2>&1
python tools/ens_rate.py 1024 16 >> gpurun_out/b128.log 2>&1
python tools/phase_times.py --config C2 --ensemble 128 >> gpurun_out/b128.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/b128_launches.csv python tools/ens_rate.py 128 2 > gpurun_out/b128_ncu.log 2>&1
