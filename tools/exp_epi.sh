timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python tools/sweep_timeline.py c5 ne 2>&1 | grep -E "chain" | head -4
TRALS_CHAIN_GEMM=1 python tools/sweep_timeline.py c5 ne 2>&1 | grep -E "chain" | head -4
for v in "" "TRALS_CHAIN_GEMM=1"; do for c in c5 c4; do echo -n "$v $c "; env $v timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"; done; done
