# round 2, fourth GPU pass: double-double R0, solvers, baseline parity (c5 NE, c4, criterion 8), QR bench lines
mkdir -p gpurun_out/r2d
timeout 600 python -m pytest tests/test_gpu_ops.py -q -k "r0 or tri or range or guard" > gpurun_out/r2d/ops.log 2>&1; echo "rc=$?" >> gpurun_out/r2d/ops.log
timeout 900 python -m pytest tests/test_gpu_solvers.py -q > gpurun_out/r2d/solvers.log 2>&1; echo "rc=$?" >> gpurun_out/r2d/solvers.log
timeout 1500 python -m pytest tests/test_gpu_baseline.py -q -k "ne or c4 or criterion8" > gpurun_out/r2d/baseline.log 2>&1; echo "rc=$?" >> gpurun_out/r2d/baseline.log
timeout 600 python tools/c4_model_probe.py > gpurun_out/r2d/c4_probe.log 2>&1
timeout 400 python bench.py --variant qr --no-cpu-baseline --no-e2e > gpurun_out/r2d/bench_c5_qr.log 2>&1
timeout 400 python bench.py --config c3 --variant qr --no-cpu-baseline --no-e2e > gpurun_out/r2d/bench_c3_qr.log 2>&1
timeout 400 python bench.py --config c2 --variant qr --no-cpu-baseline --no-e2e > gpurun_out/r2d/bench_c2_qr.log 2>&1
python tools/stability_cell.py 10 1e-10 1e-10 > gpurun_out/r2d/stability.json 2>&1
for f in ops solvers baseline; do echo "== $f"; grep -E "passed|failed|^E  |Error" gpurun_out/r2d/$f.log | head -12; done
cat gpurun_out/r2d/c4_probe.log | tail -3; tail -c 600 gpurun_out/r2d/stability.json
for f in gpurun_out/r2d/bench_*.log; do echo "== $f"; tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['config']['launch'])" 2>&1 | tail -3; done
