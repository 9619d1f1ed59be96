cd $GRAFT_REPO_ROOT
HFMM_LIB_PATH=$PWD/tools/variants/fz3.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_world.py -q -x > gpurun_out/pytest_r26_fz3.log 2>&1
for rep in 1 2; do for v in base fz3; do
  lib=base; [ $v != base ] && lib=tools/variants/$v.so
  for c in cfg4; do echo "== $v $c rep$rep"; timeout 600 python tools/variant_seq.py $lib $c 3 2>&1 | tail -1; done
done; done > gpurun_out/variants_r26.txt 2>&1
echo done
