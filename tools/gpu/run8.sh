cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py tests/test_gpu_multirank.py -q -x > gpurun_out/pytest_r8.log 2>&1
for rep in 1 2; do for v in base nofz; do
  lib=base; [ $v != base ] && lib=tools/variants/$v.so
  for c in cfg4 cfg1 cfg3; do echo "== $v $c rep$rep"; timeout 300 python tools/variant_seq.py $lib $c 3 2>&1 | tail -1; done
done; done > gpurun_out/variants_r8.txt 2>&1
python tools/prof_eval.py cfg4 1 > gpurun_out/prof_cfg4_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"_fz" -c 2 -o gpurun_out/prof_fz_cfg4 python tools/prof_eval.py cfg4 1 > gpurun_out/ncu_fz.log 2>&1
echo done
