cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r33.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py -q -x > gpurun_out/pytest_r33.log 2>&1
python bench.py --no-cpu-baseline > gpurun_out/bench_cfg4_r33.json 2> gpurun_out/bench_cfg4_r33.err
echo done
