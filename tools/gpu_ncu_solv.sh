# ncu --set full of the water-mode solvation kernel (C5 water), after a plain run exits 0
WATER=1 python tools/ens_rate.py 1024 2 > gpurun_out/plain_s.log 2>&1 && \
  WATER=1 ncu --set full --clock-control none --import-source on -k regex:"solv_group" -s 1 -c 1 \
      -o gpurun_out/solv_${TAG:-x} python tools/ens_rate.py 1024 2 > gpurun_out/ncu_s.log 2>&1
tail -1 gpurun_out/plain_s.log
