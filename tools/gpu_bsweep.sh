# C5 step by batch size (the strong-scaling floor table in DESIGN.md)
for B in 32 64 128 256 512 1024; do python tools/ens_rate.py $B 16 | sed 's/env={.*}//'; done
