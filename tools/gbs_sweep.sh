# backward-filter split model: per-SM ingest cap re-swept with 256-filter tiles (whole mesh2k_n8 step, 1 GPU)
export CUDA_VISIBLE_DEVICES=0
o=gpurun_out/gbs_sweep.txt; : > $o
for r in 1 2; do for e in "X=0" "DC_WGRAD_SM_GBS=25" "DC_WGRAD_SM_GBS=60" "DC_WGRAD_SM_GBS=100"; do
  env $e timeout 200 python bench.py --no-cpu-baseline --steps 10 --warmup 5 > gpurun_out/gbs.json 2>/dev/null
  python -c "import json,sys;d=json.loads(open('gpurun_out/gbs.json').read().strip().splitlines()[-1]);print('$e',round(d['ms_per_step'],3),d['clocks']['sm_mhz'],d['clocks']['reasons'])" >> $o
done; done
