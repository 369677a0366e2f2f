cd "${GRAFT_REPO_ROOT:-.}"
python -c "
import sys; sys.path.insert(0,'.')
from paper_2212_09005_b200 import _lib
import torch
_lib.require_cuda()
print('l2 fetch bytes now', _lib.load().fk_device_l2_fetch_bytes())
"
for L in 32 0; do
FK_L2_FETCH_BYTES=$L ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum --clock-control none -k regex:k_tcf -c 5 python scripts/prof_tcf.py 28 concurrent 2>&1 | grep -E "k_tcf|duration|dram__|lts__|l1tex" 
done
