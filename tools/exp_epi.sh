for c in c3 c4 c5; do echo "== $c"; TRALS_OZ_DBG=64 timeout 120 python tools/env_time.py $c 2 2>&1 | grep ozprof | tail -2; done
echo "== c3 W64"; TRALS_OZ_SHORT_K=1 TRALS_OZ_DBG=64 timeout 120 python tools/env_time.py c3 2 2>&1 | grep ozprof | tail -1
