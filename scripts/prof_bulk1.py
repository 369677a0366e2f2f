import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2212_09005_b200 import BulkTcf, BulkTcfParams
from paper_2212_09005_b200 import workloads as wl
p = BulkTcfParams(num_blocks=(1 << 20) // 128, seed=0)
keys = torch.from_numpy(wl.counter_stream(5, 1, int(0.9 * p.main_slots)).view(np.int64)).cuda()
for it in range(2):
    f = BulkTcf(p)
    f.insert_batch(keys)
    torch.cuda.synchronize()
