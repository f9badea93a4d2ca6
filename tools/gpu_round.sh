# GPU round script: full GPU suite + per-config benches for both fp64 engines
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu3.log
for c in c1 c2 c3 c4; do
  for e in ozaki dmma; do
    timeout 300 python bench.py --config $c --fp64-gemm $e --steps 20 --warmup 5 --no-cpu-baseline --e2e-reps 1 > gpurun_out/bench_${c}_${e}.log 2>&1
  done
done
tail -5 gpurun_out/pytest_gpu3.log
for f in gpurun_out/bench_c*_*.log; do echo $f; tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d.get('e2e',{}).get('value'))"; done
