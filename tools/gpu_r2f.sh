mkdir -p gpurun_out/r2f
timeout 600 python -m pytest tests/test_gpu_ops.py -q -k "r0 or tri or cholesky" > gpurun_out/r2f/ops.log 2>&1; echo "rc=$?" >> gpurun_out/r2f/ops.log
timeout 900 python -m pytest tests/test_gpu_solvers.py -q > gpurun_out/r2f/solvers.log 2>&1; echo "rc=$?" >> gpurun_out/r2f/solvers.log
timeout 1500 python -m pytest tests/test_gpu_baseline.py -q -k "ne or c4 or criterion8" > gpurun_out/r2f/baseline.log 2>&1; echo "rc=$?" >> gpurun_out/r2f/baseline.log
timeout 600 python tools/c4_model_probe.py > gpurun_out/r2f/c4_probe.log 2>&1
for c in c1 c2 c3 c4; do timeout 400 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/r2f/bench_$c.log 2>&1; done
timeout 400 python bench.py --variant qr --no-cpu-baseline --no-e2e > gpurun_out/r2f/bench_c5_qr.log 2>&1
timeout 400 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2f/bench_c5.log 2>&1
for f in ops solvers baseline; do echo "== $f"; grep -E "passed|failed|^E  " gpurun_out/r2f/$f.log | head -8; done
tail -2 gpurun_out/r2f/c4_probe.log
for f in gpurun_out/r2f/bench_*.log; do echo "== $f"; tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['config']['launch'])" 2>&1 | tail -2; done
