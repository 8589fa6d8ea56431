for d in ${DBG:-0 1 2 3}; do echo "debug=$d"; WSSR_OZ_DEBUG=$d PYTHONPATH=. timeout 120 python tools/ozaki_bench.py 2>&1 | grep ozaki | head -2; done
