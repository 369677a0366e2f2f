cd "${GRAFT_REPO_ROOT:-.}"
python -c "
import torch, numpy as np, sys
sys.path.insert(0,'.')
import bench
from paper_2212_09005_b200.workloads import counter_stream
a = bench.device_keys(torch, 7, bench.TAG_UNIFORM, 100000, 'cuda').cpu().numpy().view(np.uint64)
print('device_keys ok', np.array_equal(a, counter_stream(7, bench.TAG_UNIFORM, 100000)))
"
timeout 300 python bench.py --log-slots 24 --steps 3 --no-cpu --no-e2e
timeout 300 python bench.py --log-slots 28 --steps 3 --no-cpu --no-e2e
timeout 300 python bench.py --log-slots 28 --steps 3 --no-cpu --no-e2e --mode concurrent
timeout 600 python bench.py --log-slots 28 --steps 3
