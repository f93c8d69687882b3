set -u
M=gpu__time_duration.sum,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,sm__sass_inst_executed_op_global_ld.sum
for lib in paper_2208_12350_b200/libsw_b200.so build_var/libsw_code4.so; do
  SW_B200_LIB=$lib /usr/local/cuda/bin/ncu --metrics $M --clock-control none -k regex:wavefront_kernel -s 4 -c 1 --csv python tools/prof_one.py c2 2>/dev/null | grep -v "^==" > gpurun_out/r08/ncu_code4_$(basename $lib .so).csv
done
