cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_r28.log 2>&1
for rep in 1 2; do for v in base m2lv1; do
  lib=base; [ $v != base ] && lib=tools/variants/$v.so
  for c in cfg4 cfg2; do echo "== $v $c rep$rep"; timeout 300 python tools/variant_seq.py $lib $c 3 2>&1 | tail -1; done
done; done > gpurun_out/variants_r28.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_world.py tests/test_gpu_paths.py -q -x > gpurun_out/pytest_r28b.log 2>&1
echo done
