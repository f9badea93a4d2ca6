# Round profile: bench lines for every config (auto engine) + c5 with dmma, launch list of
# the default bench, one ncu --set full capture of the c5 Ozaki environment GEMM.
mkdir -p gpurun_out
for c in c1 c2 c3 c4 c5; do
  timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${c}_auto.log 2>&1
done
timeout 400 python bench.py --config c5 --variant qr --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_qr.log 2>&1
timeout 400 python bench.py --config c5 --variant qrne --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_qrne.log 2>&1
timeout 400 python bench.py --config c3 --variant qr --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_qr.log 2>&1
timeout 400 python bench.py --config c4 --dtype float32 --no-cpu-baseline > gpurun_out/bench_c4_fp32.log 2>&1
timeout 400 python bench.py --config c5 --fp64-gemm dmma --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_dmma.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5_oz.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oz8_kernel -c 1 --profile-from-start off -o gpurun_out/c5_oz64_env_bal python tools/ncu_env.py c5 ozaki > gpurun_out/ncu_full.log 2>&1
for f in gpurun_out/bench_*_auto.log gpurun_out/bench_c5_q*.log gpurun_out/bench_c3_qr.log gpurun_out/bench_c4_fp32.log gpurun_out/bench_c5_dmma.log; do
  echo "$f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value'],1), round(d['ms_per_step'],3), d['config'].get('fp64_gemm'), round(r['avg_launch_ms'],3), round(r['frac'],3), d.get('e2e',{}).get('value'))" 2>&1)"
done
