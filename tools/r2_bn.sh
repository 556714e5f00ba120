export CUDA_VISIBLE_DEVICES=0
python -m paper_1903_06681_b200.build > /dev/null
for sh in "8 64 1024 1024" "8 256 256 256" "8 512 64 64"; do timeout 120 python tools/bn_bench.py $sh; done > gpurun_out/bn_bench.txt 2>&1; cat gpurun_out/bn_bench.txt
timeout 300 ncu --set full --clock-control none -k regex:"bn_bwd|bn_apply" -c 3 -o gpurun_out/ncu_r2_bn python tools/bn_bench.py 8 64 1024 1024 --iters 1 > gpurun_out/ncu_bn.log 2>&1; echo "ncu $?"
timeout -k 10 600 python bench.py --steps 20 --warmup 5 --watchdog 500 > gpurun_out/c_bench_bf16.json 2> gpurun_out/c_bench_bf16.err; echo "bf16 $?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/c_bench_bf16.json").read().strip().splitlines()[-1])
t = {}
for l in d["config"]["layers"]:
    for k, v in l.items():
        if k.endswith("_ms") and k != "model_pred_ms":
            t[k] = round(t.get(k, 0) + v, 2)
print(round(d["value"], 1), round(d["ms_per_step"], 2), d["clocks"], t, d["roofline"]["frac"])
PY
