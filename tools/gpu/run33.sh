cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r33.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu_r33.log 2>&1
python bench.py > gpurun_out/bench_cfg4_r33.json 2> gpurun_out/bench_cfg4_r33.err
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref_r33.json 2> gpurun_out/bench_ref_r33.err
for c in cfg2 cfg3 cfg5; do python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${c}_r33.json 2> gpurun_out/bench_${c}_r33.err; done
python tools/prof_eval.py cfg4 1 > gpurun_out/prof_cfg4_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_cfg4_r33.csv python tools/prof_eval.py cfg4 1 > gpurun_out/ncu_cfg4_r33.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_m2l_dmma|_fz2|k_l2l_theta_rb|k_l2l_phi_rb|k_m2m_theta_rbl|k_l2l_theta_rbl" -c 14 -o gpurun_out/prof_r33_cfg4 python tools/prof_eval.py cfg4 1 > gpurun_out/ncu_r33.log 2>&1
echo done
