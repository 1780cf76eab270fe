M=gpu__time_duration.sum,l1tex__m_l1tex2xbar_req_cycles_active.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_sectors.sum,lts__t_requests_srcunit_tex.sum,lts__t_sectors_srcunit_tex.sum,sm__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_tex_mem_texture.sum,l1tex__t_sectors_pipe_tex_mem_texture.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_tex_wavefronts.sum,l1tex__m_l1tex2xbar_req.sum
for v in base lp1 lp1_tex0; do
HRT_LIB=tools/_variants/libhrt_$v.so ncu --metrics $M --clock-control none -k regex:k_field_ws -s 3 -c 1 --csv python tools/quick_bench.py 1 800x800 1 1 > gpurun_out/ncu_$v.csv 2>&1
done
