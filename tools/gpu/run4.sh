cd $GRAFT_REPO_ROOT
timeout 600 python tools/leaf_ab.py cfg4 HFMM_L2T_V2 5 > gpurun_out/ab_l2t_cfg4.txt 2>&1
timeout 600 python tools/leaf_ab.py cfg2 HFMM_L2T_V2 5 > gpurun_out/ab_l2t_cfg2.txt 2>&1
timeout 600 python tools/leaf_ab.py cfg5 HFMM_L2T_V2 3 > gpurun_out/ab_l2t_cfg5.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py tests/test_gpu_adapter.py -q -x > gpurun_out/pytest_r4.log 2>&1
python tools/prof_eval.py cfg4 1 > gpurun_out/prof_cfg4_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_c2m_quad2|k_l2t_quad3" -c 2 -o gpurun_out/prof_leaf2_cfg4 python tools/prof_eval.py cfg4 1 > gpurun_out/ncu_leaf2.log 2>&1
echo done
