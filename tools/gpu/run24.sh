cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py tests/test_gpu_world.py tests/test_gpu_multirank.py -q -x > gpurun_out/pytest_r24.log 2>&1
for rep in 1 2; do for v in base fzl; do
  lib=base; [ $v != base ] && lib=tools/variants/$v.so
  for c in cfg4 cfg2; do echo "== $v $c rep$rep"; timeout 600 python tools/variant_seq.py $lib $c 3 2>&1 | tail -1; done
done; done > gpurun_out/variants_r24.txt 2>&1
HFMM_LIB_PATH=$PWD/tools/variants/fzl.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_r24_fzl.log 2>&1
echo done
