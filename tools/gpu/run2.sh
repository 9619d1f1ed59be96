cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_paths.py tests/test_full_configs.py -q -rs -s > gpurun_out/pytest_r2.log 2>&1
timeout 300 python bench.py --force-dist --steps 3 --warmup 3 --config cfg2 > gpurun_out/bench_forcedist.json 2> gpurun_out/bench_forcedist.err
timeout 900 python tools/rank_scaling.py cfg2 1 2 4 8 > gpurun_out/rank_scaling_cfg2.txt 2>&1
timeout 900 python tools/rank_scaling.py cfg3 1 2 4 8 > gpurun_out/rank_scaling_cfg3.txt 2>&1
echo done
