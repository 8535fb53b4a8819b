# ncu --set full of the cluster pair kernel only (C5), after a plain run exits 0
python tools/ens_rate.py 1024 4 > gpurun_out/plain_p.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"cluster_pair" -s 2 -c 1 \
      -o gpurun_out/pair_${TAG:-x} python tools/ens_rate.py 1024 4 > gpurun_out/ncu_p.log 2>&1
tail -2 gpurun_out/plain_p.log
