import sys, json, argparse
sys.path.insert(0, ".")
import bench
r = bench.measure_producer("c1", argparse.Namespace())
print(json.dumps(r, indent=1))
