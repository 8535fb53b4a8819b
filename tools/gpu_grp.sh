# 32-octet group-box skip (cur) vs without (nogrp): parity + C5 A/B + B = 128
python -m pytest tests/test_gpu_bench_parity.py tests/test_gpu_parity.py -x -q 2>&1 | tail -1
bash tools/ab.sh 1024 16 cur nogrp 2>&1 | sed 's/env={.*}//'
bash tools/ab.sh 128 16 cur nogrp 2>&1 | sed 's/env={.*}//'
