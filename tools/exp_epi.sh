timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python tools/sweep_timeline.py c5 ne 2>&1 | grep -E "solve|chol|S[0-9]" | head -12
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"
