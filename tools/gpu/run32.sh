cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_paths.py -q -x -k "leaf_m2l or natural" > gpurun_out/pytest_r32.log 2>&1
python bench.py --no-cpu-baseline > gpurun_out/bench_cfg4_r32.json 2> gpurun_out/bench_cfg4_r32.err
python bench.py --config cfg2 --no-cpu-baseline > gpurun_out/bench_cfg2_r32.json 2> gpurun_out/bench_cfg2_r32.err
echo done
