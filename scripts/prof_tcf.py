"""One pass of each point-TCF op at 2^28 slots, for ncu captures (not a bench)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2212_09005_b200 import Tcf

log_slots = int(sys.argv[1]) if len(sys.argv) > 1 else 28
mode = sys.argv[2] if len(sys.argv) > 2 else "ordered"
g = int(sys.argv[3]) if len(sys.argv) > 3 else 1
n = int(0.9 * (1 << log_slots))
keys = bench.device_keys(torch, 1, bench.TAG_UNIFORM, n, "cuda")
negs = bench.device_keys(torch, 2, bench.TAG_FPR, n, "cuda")
f = Tcf(num_blocks=(1 << log_slots) // 16, mode=mode, group_width=g)
f.insert_many(keys)
f.query_many(keys)
f.query_many(negs)
f.delete_many(keys)
torch.cuda.synchronize()
print("done")
