# round 2, third GPU pass: R0 / guard operators, solvers, 2-process shard test, c5 NE + c4 baselines,
# QR bench lines at c3 and c5
mkdir -p gpurun_out/r2c
timeout 600 python -m pytest tests/test_gpu_ops.py -q -k "r0 or tri or range or guard or core_householder" > gpurun_out/r2c/ops.log 2>&1; echo "rc=$?" >> gpurun_out/r2c/ops.log
timeout 900 python -m pytest tests/test_gpu_solvers.py -q -x > gpurun_out/r2c/solvers.log 2>&1; echo "rc=$?" >> gpurun_out/r2c/solvers.log
timeout 1200 python -m pytest tests/test_gpu_shard.py -q > gpurun_out/r2c/shard.log 2>&1; echo "rc=$?" >> gpurun_out/r2c/shard.log
timeout 1500 python -m pytest tests/test_gpu_baseline.py -q -k "ne or c4 or criterion8" --durations=10 > gpurun_out/r2c/baseline.log 2>&1; echo "rc=$?" >> gpurun_out/r2c/baseline.log
timeout 400 python bench.py --variant qr --no-cpu-baseline --no-e2e > gpurun_out/r2c/bench_c5_qr.log 2>&1
timeout 400 python bench.py --config c3 --variant qr --no-cpu-baseline --no-e2e > gpurun_out/r2c/bench_c3_qr.log 2>&1
for f in ops solvers shard baseline; do echo "== $f"; tail -12 gpurun_out/r2c/$f.log; done
for f in gpurun_out/r2c/bench_*.log; do echo "== $f"; tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['config']['launch'])" 2>&1 | tail -3; done
