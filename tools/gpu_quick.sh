# quick GPU check: Ozaki operator tests + c5 bench
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_ops.py -q -k "oz" > gpurun_out/oz_tests.log 2>&1; echo "rc=$?" >> gpurun_out/oz_tests.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_quick.log 2>&1
tail -3 gpurun_out/oz_tests.log
tail -1 gpurun_out/bench_quick.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('sweeps/s', d['value'], 'ms', d['ms_per_step'], 'env ms', r['avg_launch_ms'], 'frac', r['frac'], 'e2e', d.get('e2e',{}).get('value'), 'xdig', d['config'].get('x_digits_ms'), 'err', d['final_error'])"
