cd "${GRAFT_REPO_ROOT:-.}"
./scripts/micro/gather
./scripts/micro/gather 32 | head -3
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum --clock-control none -k regex:gather -s 1 -c 1 ./scripts/micro/gather 2>&1 | grep -E "dram|lts|l1tex|duration|gather<"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum --clock-control none -k regex:gather -s 13 -c 1 ./scripts/micro/gather 2>&1 | grep -E "dram|lts|l1tex|duration|gather<"
