cd $GRAFT_REPO_ROOT
python tools/prof_eval.py cfg4 1 > gpurun_out/prof_cfg4_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_p2p" -c 2 -o gpurun_out/prof_p2p_cfg4 python tools/prof_eval.py cfg4 1 > gpurun_out/ncu_p2p.log 2>&1
nproc > gpurun_out/ref_host.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/ref_host.txt
timeout 600 python tools/ref_full_time.py cfg2 gpurun_out/r02_ref_full_cfg2.json > gpurun_out/ref_full_cfg2.log 2>&1
timeout 1800 python tools/ref_full_time.py cfg4 gpurun_out/r02_ref_full_cfg4.json > gpurun_out/ref_full_cfg4.log 2>&1
echo done
