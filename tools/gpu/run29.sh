cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r29.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu_r29.log 2>&1
python bench.py > gpurun_out/bench_cfg4_r29.json 2> gpurun_out/bench_cfg4_r29.err
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref_r29.json 2> gpurun_out/bench_ref_r29.err
echo done
