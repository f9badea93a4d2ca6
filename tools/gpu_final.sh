# End-of-round measurement: GPU suite, smoke, every config's bench line, c5 variants, the
# reference arm, the c5 launch list and one ncu --set full of the dominant kernel.
mkdir -p gpurun_out/final
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1
timeout 400 python bench.py > gpurun_out/final/bench_default.log 2>&1
for c in c1 c2 c3 c4; do timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/final/bench_$c.log 2>&1; done
for v in qr qrne; do timeout 400 python bench.py --variant $v --no-cpu-baseline --no-e2e > gpurun_out/final/bench_c5_$v.log 2>&1; done
timeout 400 python bench.py --config c2 --variant qr --no-cpu-baseline --no-e2e > gpurun_out/final/bench_c2_qr.log 2>&1
timeout 400 python bench.py --config c3 --variant qr --no-cpu-baseline --no-e2e > gpurun_out/final/bench_c3_qr.log 2>&1
timeout 400 python bench.py --config c4 --dtype float32 --no-cpu-baseline > gpurun_out/final/bench_c4_fp32.log 2>&1
timeout 400 python bench.py --fp64-gemm dmma --no-cpu-baseline --no-e2e > gpurun_out/final/bench_c5_dmma.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/bench_ref.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/final/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --eager > gpurun_out/final/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oz8_kernel -c 1 --profile-from-start off -f -o gpurun_out/final/c5_oz64_env python tools/ncu_env.py c5 ozaki > gpurun_out/final/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oz8_kernel -c 1 --profile-from-start off -f -o gpurun_out/final/c3_oz64_env python tools/ncu_env.py c3 ozaki > gpurun_out/final/ncu_full_c3.log 2>&1
tail -1 gpurun_out/final/pytest_gpu.log; tail -1 gpurun_out/final/smoke.log
for f in gpurun_out/final/bench_*.log; do echo "$f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(round(d['value'],2), round(d['ms_per_step'],3), d['config'].get('fp64_gemm'), r.get('avg_launch_ms'), r.get('frac'), d.get('e2e',{}).get('value'))" 2>&1)"; done
