# round 2, first GPU pass: GPU suite + smoke, the reworked bench (default c5 line with the
# full-sweep CPU baseline and the default-config e2e), the reference arm (full-size block updates)
# and the host facts of the box
mkdir -p gpurun_out/r2a
(nproc; lscpu | head -20; free -g; nvidia-smi -L) > gpurun_out/r2a/host.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2a/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2a/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a/smoke.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a/bench_default.log 2>&1
timeout 900 python bench.py --impl reference --steps 4 --warmup 1 > gpurun_out/r2a/bench_ref.log 2>&1
tail -2 gpurun_out/r2a/pytest_gpu.log; tail -1 gpurun_out/r2a/smoke.log
tail -c 3000 gpurun_out/r2a/bench_default.log; tail -c 2500 gpurun_out/r2a/bench_ref.log
