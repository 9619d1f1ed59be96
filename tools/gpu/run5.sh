cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for v in base ob4 ob2mb4 ob4mb3 ob1; do
  lib=paper_2006_15367_b200/_lib/libhfmm_b200.so; [ $v != base ] && lib=tools/variants/$v.so
  for c in cfg4 cfg2; do echo "== $v $c rep$rep"; timeout 300 python tools/variant_eval.py $lib $c 3 2>&1 | tail -1; done
done; done > gpurun_out/l2t_variants.txt 2>&1
echo done
