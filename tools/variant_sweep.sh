# A/B of prebuilt library variants (paper_2006_15367_b200/_lib/variants/*.so) through bench.py.
mkdir -p gpurun_out
for rep in 1 2; do
for v in base l2lc5 l2lc8 ug4; do
  echo "== $v rep$rep"
  HFMM_LIB_PATH=paper_2006_15367_b200/_lib/variants/$v.so python bench.py --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['phase_ms'].items()})"
done; done > gpurun_out/vsweep.log 2>&1
cat gpurun_out/vsweep.log
