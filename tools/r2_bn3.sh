export CUDA_VISIBLE_DEVICES=0
python -m paper_1903_06681_b200.build > /dev/null
timeout -k 10 900 python -m pytest tests/test_gpu_network.py tests/test_pool.py tests/test_gpu_fp32.py -m gpu -q -x > gpurun_out/d_tests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/d_tests.log
for sh in "8 64 1024 1024" "8 256 256 256" "8 512 64 64"; do timeout 120 python tools/bn_bench.py $sh; done
timeout -k 10 600 python bench.py --workload mesh2k_n8_net --steps 10 --warmup 5 --no-cpu-baseline --watchdog 500 > gpurun_out/d_bench_net.json 2> gpurun_out/d_bench_net.err; echo "net $?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/d_bench_net.json").read().strip().splitlines()[-1])
t = {}
for l in d["config"]["layers"]:
    for k, v in l.items():
        if k.endswith("_ms") and k != "model_pred_ms":
            t[k] = round(t.get(k, 0) + v, 2)
print(round(d["value"], 1), round(d["ms_per_step"], 2), d["clocks"]["sm_mhz"], t)
PY
