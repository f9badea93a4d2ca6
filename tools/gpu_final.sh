# End-of-round measurement: GPU suite, smoke, every config's bench line, c5 variants and engines,
# the reference arm, the c5 launch list and one ncu --set full of the dominant kernel.
# usage: bash tools/gpu_final.sh [tag]
T=gpurun_out/${1:-final}; mkdir -p $T
(nproc; lscpu | head -20; free -g; nvidia-smi -L) > $T/host.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=15 > $T/pytest_gpu.log 2>&1; echo "rc=$?" >> $T/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $T/smoke.log 2>&1
timeout 900 python bench.py > $T/bench_default.log 2>&1
for c in c1 c2 c3 c4; do timeout 400 python bench.py --config $c --no-cpu-baseline > $T/bench_$c.log 2>&1; done
for v in qr qrne; do timeout 400 python bench.py --variant $v --no-cpu-baseline --no-e2e > $T/bench_c5_$v.log 2>&1; done
timeout 400 python bench.py --config c2 --variant qr --no-cpu-baseline --no-e2e > $T/bench_c2_qr.log 2>&1
timeout 400 python bench.py --config c3 --variant qr --no-cpu-baseline --no-e2e > $T/bench_c3_qr.log 2>&1
timeout 400 python bench.py --config c4 --dtype float32 --no-cpu-baseline > $T/bench_c4_fp32.log 2>&1
timeout 400 python bench.py --fp64-gemm ozaki --no-cpu-baseline --no-e2e > $T/bench_c5_ozaki.log 2>&1
timeout 400 python bench.py --fp64-gemm dmma --no-cpu-baseline --no-e2e > $T/bench_c5_dmma.log 2>&1
TRALS_CRT_MODULI=16 timeout 400 python bench.py --no-cpu-baseline --no-e2e > $T/bench_c5_crt16.log 2>&1
timeout 900 python bench.py --impl reference --steps 4 --warmup 1 > $T/bench_ref.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 700 --csv --log-file $T/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --eager > $T/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:crt8_kernel -c 1 -f -o $T/c5_crt_env python tools/env_bench.py --engines crt --reps 1 > $T/ncu_full.log 2>&1
ncu -i $T/c5_crt_env.ncu-rep --page raw --csv > $T/c5_crt_env_raw.csv 2>/dev/null
timeout 200 python tools/env_bench.py --engines crt,oz64,dmma > $T/env_bench.log 2>&1
timeout 200 python tools/ncu_res.py c5 time > $T/res_time.log 2>&1
timeout 200 python tools/chol_prof.py > $T/chol_time.log 2>&1
grep -E "passed|failed" $T/pytest_gpu.log | tail -2; tail -1 $T/smoke.log
for f in $T/bench_*.log; do echo "$f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print(round(d['value'],4), round(d['ms_per_step'],3), d['config'].get('fp64_gemm'), r.get('avg_launch_ms'), r.get('frac'), d.get('e2e',{}).get('value'))" 2>&1)"; done
cat $T/env_bench.log $T/res_time.log $T/chol_time.log | tail -12
