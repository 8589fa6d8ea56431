for m in 8 13 14; do echo "mode $m"; OZ_TRACE_MODE=$m PYTHONPATH=. timeout 60 python tools/ozaki_timeline.py 1 | sed -n '10,13p;$p'; done
for m in 0 5 6; do echo "bench mode $m"; WSSR_OZ_DEBUG=$m PYTHONPATH=. timeout 60 python tools/ozaki_bench.py --one | tail -1; done
