mkdir -p gpurun_out/r2g
timeout 600 python -m pytest tests/test_gpu_ops.py -q -k "refine or cholesky or r0 or tri" > gpurun_out/r2g/ops.log 2>&1; echo "rc=$?" >> gpurun_out/r2g/ops.log
timeout 900 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_ring_api.py -q > gpurun_out/r2g/solvers.log 2>&1; echo "rc=$?" >> gpurun_out/r2g/solvers.log
timeout 1500 python -m pytest tests/test_gpu_baseline.py -q > gpurun_out/r2g/baseline.log 2>&1; echo "rc=$?" >> gpurun_out/r2g/baseline.log
for c in c1 c2 c3 c4; do timeout 400 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/r2g/bench_$c.log 2>&1; done
timeout 400 python bench.py --config c2 --variant qr --no-cpu-baseline --no-e2e > gpurun_out/r2g/bench_c2_qr.log 2>&1
for f in ops solvers baseline; do echo "== $f"; grep -E "passed|failed|^E  " gpurun_out/r2g/$f.log | head -8; done
for f in gpurun_out/r2g/bench_*.log; do echo "== $f"; tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['config']['launch'])" 2>&1 | tail -2; done
