"""Kernel launches of one decode-time index update (ClusterIndex.update) of
128 units: run under ncu; the update's k-means launches are the last ones."""
import argparse, json, sys
sys.path.insert(0, ".")
import torch
import bench
a = argparse.Namespace(batch=16, ctx=16384)
print(json.dumps(bench.run_update_cost(a, torch, torch.device("cuda"), print)))
