python tools/chol_time.py 400; TRALS_CHOL_UNFUSED=1 python tools/chol_time.py 400
timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/chol_fused.csv -k regex:chol python tools/chol_time.py 400 > /dev/null 2>&1
