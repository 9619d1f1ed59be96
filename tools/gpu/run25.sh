cd $GRAFT_REPO_ROOT
python tools/prof_eval.py cfg4 1 > gpurun_out/prof_cfg4_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"_fz2|k_l2l_theta_rb|k_l2l_phi_rb" -c 6 -o gpurun_out/prof_r25_cfg4 python tools/prof_eval.py cfg4 1 > gpurun_out/ncu_r25.log 2>&1
echo done
