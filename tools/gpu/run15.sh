cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r15.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rs -x > gpurun_out/pytest_gpu_r15.log 2>&1
python bench.py > gpurun_out/bench_cfg4_r15.json 2> gpurun_out/bench_cfg4_r15.err
python bench.py --config cfg2 > gpurun_out/bench_cfg2_r15.json 2> gpurun_out/bench_cfg2_r15.err
echo done
