# FK phase clocks of CTA 0 (FK_TIMING build) at one CTA per SM and at the bench batch
for B in 148 1024; do KFB200_LIB=$PWD/_variants/fkt.so python tools/phase_times.py --ensemble $B --iters 6 2>&1 | grep FKT | tail -2; done
