# whole-step A/B of existing switches at HEAD (mesh2k_n8, 1 B200): PDL off, 128-wide forward N tiles, fused multi-tile BN
export CUDA_VISIBLE_DEVICES=0
o=gpurun_out/knob_step_ab.txt; : > $o
for r in 1 2; do for e in "X=0" "DC_NO_PDL=1" "DC_V2_BN=128" "DC_BN_FUSE_NT=1"; do
  env $e timeout 200 python bench.py --no-cpu-baseline --steps 10 --warmup 5 > gpurun_out/gbs.json 2>/dev/null
  python -c "import json,sys;d=json.loads(open('gpurun_out/gbs.json').read().strip().splitlines()[-1]);print('$e',round(d['ms_per_step'],3),d['clocks']['sm_mhz'],d['clocks']['reasons'])" >> $o
done; done
