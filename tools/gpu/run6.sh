cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for v in base ob1mb5 ob2 p2pold lw128 lw64; do
  lib=base; [ $v != base ] && lib=tools/variants/$v.so
  for c in cfg4 cfg2 cfg3; do echo "== $v $c rep$rep"; timeout 300 python tools/variant_seq.py $lib $c 3 2>&1 | tail -1; done
done; done > gpurun_out/variants_r6.txt 2>&1
echo done
