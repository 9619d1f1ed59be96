cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_r31.log 2>&1
python bench.py > gpurun_out/bench_cfg4_r31.json 2> gpurun_out/bench_cfg4_r31.err
python bench.py --config cfg2 --no-cpu-baseline > gpurun_out/bench_cfg2_r31.json 2> gpurun_out/bench_cfg2_r31.err
echo done
