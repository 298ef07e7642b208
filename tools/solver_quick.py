import sys, json, os
sys.path.insert(0, os.getcwd())
import bench
print(json.dumps(bench.solver_bench()))
