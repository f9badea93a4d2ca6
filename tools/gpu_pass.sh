# One GPU pass: GPU suite, smoke, default bench line + reference arm, c5 launch list.
# usage: bash tools/gpu_pass.sh <tag> [pytest -k expr]
T=gpurun_out/$1; mkdir -p $T
(nproc; lscpu | head -20; free -g; nvidia-smi -L) > $T/host.txt 2>&1
if [ -n "$2" ]; then K="-k $2"; else K=""; fi
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=25 $K > $T/pytest_gpu.log 2>&1; echo "rc=$?" >> $T/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $T/smoke.log 2>&1
timeout 900 python bench.py > $T/bench_default.log 2>&1
timeout 900 python bench.py --impl reference --steps 4 --warmup 1 > $T/bench_ref.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file $T/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --eager > $T/ncu_launch.log 2>&1
grep -E "passed|failed" $T/pytest_gpu.log | tail -3; grep -E "^FAILED|^ERROR" $T/pytest_gpu.log | head -20; tail -1 $T/smoke.log
tail -c 2500 $T/bench_default.log; echo; tail -c 2000 $T/bench_ref.log
