cd $GRAFT_REPO_ROOT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
for c in cfg3 cfg5; do
  timeout 600 python tools/prof_eval.py $c 1 > gpurun_out/prof_${c}_plain_r34.log 2>&1 && \
  timeout 1500 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_${c}_r34.csv python tools/prof_eval.py $c 1 > gpurun_out/ncu_${c}_r34.log 2>&1
done
echo done
