cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py tests/test_gpu_world.py -q -x > gpurun_out/pytest_r18.log 2>&1
for rep in 1 2; do for v in base nofzl; do
  lib=base; [ $v != base ] && lib=tools/variants/$v.so
  for c in cfg4 cfg2; do echo "== $v $c rep$rep"; timeout 300 python tools/variant_seq.py $lib $c 3 2>&1 | tail -1; done
done; done > gpurun_out/variants_r18.txt 2>&1
python tools/prof_eval.py cfg4 1 > gpurun_out/prof_cfg4_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_m2l_dmma|_fz2|k_c2m|k_l2t|k_p2p_leaf2" -c 10 -o gpurun_out/prof_r18_cfg4 python tools/prof_eval.py cfg4 1 > gpurun_out/ncu_r18.log 2>&1
echo done
