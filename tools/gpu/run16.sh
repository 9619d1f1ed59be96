cd $GRAFT_REPO_ROOT
python tools/prof_eval.py cfg4 1 > gpurun_out/prof_cfg4_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_cfg4_r16.csv python tools/prof_eval.py cfg4 1 > gpurun_out/ncu_cfg4_r16.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_m2m_fz|k_l2l_theta_rb|k_m2m_theta_rbl|k_l2l_phi_rb" -c 20 -o gpurun_out/prof_interp_cfg4 python tools/prof_eval.py cfg4 1 > gpurun_out/ncu_interp.log 2>&1
echo done
