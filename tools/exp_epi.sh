timeout 300 python -m pytest tests/test_gpu_ops.py -q -x -k "oz" 2>&1 | tail -1
for c in c5 c3 c4; do timeout 120 python tools/env_time.py $c 5 2>&1 | tail -1; done
