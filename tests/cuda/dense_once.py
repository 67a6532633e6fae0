import sys, types
sys.path.insert(0, "/root/repo")
import bench
args = types.SimpleNamespace(steps=2, warmup=3)
print(bench.run_dense(args, 0, 1, 0)["tokens_per_s"])
