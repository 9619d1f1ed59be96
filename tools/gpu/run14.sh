cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r14.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu_r14.log 2>&1
python bench.py > gpurun_out/bench_cfg4_r14.json 2> gpurun_out/bench_cfg4_r14.err
timeout 1200 python tools/rank_scaling.py cfg4 1 2 4 8 > gpurun_out/rank_scaling_cfg4.txt 2>&1
timeout 600 python tools/rank_scaling.py cfg2 1 2 4 8 > gpurun_out/rank_scaling_cfg2.txt 2>&1
python tools/prof_eval.py cfg4 1 > gpurun_out/prof_cfg4_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_cfg4_r14.csv python tools/prof_eval.py cfg4 1 > gpurun_out/ncu_cfg4_r14.log 2>&1
echo done
