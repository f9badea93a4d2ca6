# round 2, fifth GPU pass: operator fixes + the reference API helpers, the exact-error residual
# (timing + one ncu --set full capture), compute-sanitizer on the int8 kernels
mkdir -p gpurun_out/r2e
timeout 600 python -m pytest tests/test_gpu_ops.py -q -k "r0 or tri or cholesky" > gpurun_out/r2e/ops.log 2>&1; echo "rc=$?" >> gpurun_out/r2e/ops.log
timeout 600 python -m pytest tests/test_gpu_ring_api.py -q > gpurun_out/r2e/ring_api.log 2>&1; echo "rc=$?" >> gpurun_out/r2e/ring_api.log
timeout 300 python tools/ncu_res.py c5 time > gpurun_out/r2e/res_time.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oz8_kernel -c 1 --profile-from-start off -f -o gpurun_out/r2e/c5_residual python tools/ncu_res.py c5 profile > gpurun_out/r2e/ncu_res.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_ops.py -q -x -k "test_env_oz64_matches_f64 and 300-77 or test_env_oz64_deterministic or test_env_oz_matches_f64 and 300-77" > gpurun_out/r2e/sanitizer_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/r2e/sanitizer_$tool.log
done
for f in ops ring_api; do echo "== $f"; grep -E "passed|failed|^E  " gpurun_out/r2e/$f.log | head -10; done
cat gpurun_out/r2e/res_time.log | tail -2; tail -3 gpurun_out/r2e/ncu_res.log
for tool in memcheck racecheck synccheck; do echo "== $tool"; grep -E "ERROR SUMMARY|passed|failed|rc=" gpurun_out/r2e/sanitizer_$tool.log | tail -4; done
