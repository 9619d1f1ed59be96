cd $GRAFT_REPO_ROOT
for rep in 1 2; do for v in base nofz m2monly; do
  lib=base; [ $v != base ] && lib=tools/variants/$v.so
  for c in cfg4 cfg3; do echo "== $v $c rep$rep"; timeout 300 python tools/variant_seq.py $lib $c 3 2>&1 | tail -1; done
done; done > gpurun_out/variants_r10.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "phase_by_phase" > gpurun_out/pytest_r10.log 2>&1
echo done
