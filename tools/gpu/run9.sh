cd $GRAFT_REPO_ROOT
for rep in 1 2; do for v in base nofz; do
  lib=base; [ $v != base ] && lib=tools/variants/$v.so
  for c in cfg4 cfg2; do echo "== $v $c rep$rep"; timeout 300 python tools/variant_seq.py $lib $c 3 2>&1 | tail -1; done
done; done > gpurun_out/variants_r9.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_configs.py -q -x -s -k "phase_by_phase or golden or full_config" > gpurun_out/pytest_r9.log 2>&1
echo done
