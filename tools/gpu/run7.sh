cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu_r7.log 2>&1
python bench.py > gpurun_out/bench_cfg4_r7.json 2> gpurun_out/bench_cfg4_r7.err
for c in cfg2 cfg3 cfg5; do python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${c}_r7.json 2>&1; done
echo done
