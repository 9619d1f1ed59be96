cd $GRAFT_REPO_ROOT
for c in cfg3 cfg5 cfg1; do
  timeout 600 python tools/variant_check.py base $c 3 2>&1 | tail -1
  for v in blk0 blk15; do timeout 600 python tools/variant_check.py tools/variants/$v.so $c 3 2>&1 | tail -1; done
done > gpurun_out/variants_r30.txt 2>&1
rm -f gpurun_out/_pot_*.npy
echo done
