# GPU check after a numerics change: full GPU suite, smoke, c5/c3/c4 benches (no CPU baseline)
mkdir -p gpurun_out/check
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/check/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/check/pytest_gpu.log
tail -3 gpurun_out/check/pytest_gpu.log
for c in c5 c3 c4; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/check/bench_$c.log 2>&1
  tail -1 gpurun_out/check/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$c', 'sweeps/s', d['value'], 'ms', d['ms_per_step'], 'env ms', r['avg_launch_ms'], 'frac', r['frac'], 'e2e', d.get('e2e',{}).get('value'), 'err', d.get('final_error'), d.get('clocks'))"
done
