# torque-step phase clocks of CTA 0 (TQ_TIMING build) at one CTA per SM and at the bench batch
for B in 148 1024; do KFB200_LIB=$PWD/_variants/tqt.so python tools/phase_times.py --ensemble $B --iters 6 2>&1 | grep TQT | tail -2; done
