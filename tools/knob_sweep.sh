mkdir -p gpurun_out
run() { echo "== $*"; env "$@" python bench.py --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['phase_ms'].items()})"; }
{
run X=0
run HFMM_BIG_THREADS=128
run HFMM_BIG_THREADS=512
run HFMM_PHI_CTAS=3
run HFMM_PHI_CTAS=4
run HFMM_C2M_RMAX=2
run HFMM_C2M_RMAX=8
run X=1
for c in cfg3 cfg4; do echo "== $c"; python bench.py --no-cpu-baseline --config $c --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3))"; echo "== $c threads512"; HFMM_BIG_THREADS=512 python bench.py --no-cpu-baseline --config $c --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3))"; done
} > gpurun_out/sweep.log 2>&1
cat gpurun_out/sweep.log
