cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py tests/test_gpu_world.py tests/test_gpu_multirank.py tests/test_gpu_adapter.py -q -x > gpurun_out/pytest_r29.log 2>&1
for rep in 1 2; do for v in base; do
  lib=base; [ $v != base ] && lib=tools/variants/$v.so
  for c in cfg4 cfg2 cfg3; do echo "== $v $c rep$rep"; timeout 300 python tools/variant_seq.py $lib $c 3 2>&1 | tail -1; done
done; done > gpurun_out/variants_r29.txt 2>&1
echo done
