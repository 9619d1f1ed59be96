cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_world.py tests/test_setup_import.py tests/test_gpu_multirank.py -q -rs -m gpu > gpurun_out/pytest_r3.log 2>&1
PYTHONFAULTHANDLER=1 timeout -s ABRT 240 python bench.py --force-dist --steps 3 --warmup 3 --config cfg2 --no-cpu-baseline > gpurun_out/bench_forcedist.json 2> gpurun_out/bench_forcedist.err
timeout 900 python tools/rank_scaling.py cfg3 1 2 4 8 > gpurun_out/rank_scaling_cfg3.txt 2>&1
python tools/prof_eval.py cfg4 1 > gpurun_out/prof_cfg4_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_c2m_quad2|k_l2t_quad2|k_m2m_theta_rb|k_l2l_theta_rb" -c 4 -o gpurun_out/prof_leaf_cfg4 python tools/prof_eval.py cfg4 1 > gpurun_out/ncu_leaf.log 2>&1
echo done
