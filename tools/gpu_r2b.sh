# round 2, second GPU pass: the merged-R0 QR path (operator + solver tests), the c5 bench line
mkdir -p gpurun_out/r2b
timeout 600 python -m pytest tests/test_gpu_ops.py -q -k "r0 or tri" > gpurun_out/r2b/ops_r0.log 2>&1; echo "rc=$?" >> gpurun_out/r2b/ops_r0.log
timeout 900 python -m pytest tests/test_gpu_solvers.py -q > gpurun_out/r2b/solvers.log 2>&1; echo "rc=$?" >> gpurun_out/r2b/solvers.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2b/bench_default.log 2>&1
timeout 400 python bench.py --variant qr --no-cpu-baseline --no-e2e > gpurun_out/r2b/bench_c5_qr.log 2>&1
timeout 400 python bench.py --config c3 --variant qr --no-cpu-baseline --no-e2e > gpurun_out/r2b/bench_c3_qr.log 2>&1
tail -5 gpurun_out/r2b/ops_r0.log; tail -5 gpurun_out/r2b/solvers.log
for f in gpurun_out/r2b/bench_*.log; do echo "== $f"; tail -c 1500 $f; echo; done
