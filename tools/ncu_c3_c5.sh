# ncu --set full of one environment GEMM launch at c3 and c4 (after a plain run)
mkdir -p gpurun_out/prof
python tools/ncu_env.py c3 ozaki > gpurun_out/prof/plain_c3.log 2>&1; echo "plain rc=$?"
for c in c3 c4; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oz8_kernel -c 1 --profile-from-start off -o gpurun_out/prof/${c}_env -f python tools/ncu_env.py $c ozaki > gpurun_out/prof/ncu_$c.log 2>&1; echo "ncu $c rc=$?"
done
