# FK / torque phase clocks of CTA 0 for a single trajectory and B = 64
for B in 1 64; do
  KFB200_LIB=$PWD/_variants/fkt.so python tools/phase_times.py --ensemble $B --iters 6 2>&1 | grep FKT | tail -2 | sed "s/^/B=$B /"
  KFB200_LIB=$PWD/_variants/tqt.so python tools/phase_times.py --ensemble $B --iters 6 2>&1 | grep TQT | tail -2 | sed "s/^/B=$B /"
done
