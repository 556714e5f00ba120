# 1-GPU: BN-kernel validation, fused-BN-statistics A/B per layer, bench lines
export CUDA_VISIBLE_DEVICES=0
python -m paper_1903_06681_b200.build > /dev/null
timeout -k 10 900 python -m pytest tests/test_gpu_network.py tests/test_pool.py tests/test_gpu_conv.py tests/test_loopback.py -m gpu -q -x > gpurun_out/a_tests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/a_tests.log
for sh in "8 64 1024 1024 64 3 1 1" "8 128 512 512 128 3 1 1" "8 64 1024 1024 128 3 2 1" "8 128 512 512 256 3 2 1" "8 256 256 256 256 3 1 1" "8 512 128 128 512 3 1 1" "8 512 64 64 512 3 1 1"; do
  for f in "" "--bn-fused"; do
    echo "== $sh $f"; timeout 120 python tools/kbench.py $sh --ops fwd --iters 20 --warmup 5 --flush $f 2>&1 | tail -1
  done
done > gpurun_out/a_bnfuse_ab.txt; cat gpurun_out/a_bnfuse_ab.txt
timeout -k 10 600 python bench.py --steps 20 --warmup 5 --watchdog 500 > gpurun_out/a_bench_bf16.json 2> gpurun_out/a_bench_bf16.err; echo "bf16 $?"
timeout -k 10 600 python bench.py --workload mesh2k_n8_net --steps 10 --warmup 5 --no-cpu-baseline --watchdog 500 > gpurun_out/a_bench_net.json 2> gpurun_out/a_bench_net.err; echo "net $?"
python - <<'PY'
import json
for f in ("a_bench_bf16", "a_bench_net"):
    d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
    t = {}
    for l in d["config"]["layers"]:
        for k, v in l.items():
            if k.endswith("_ms") and k != "model_pred_ms":
                t[k] = round(t.get(k, 0) + v, 2)
    print(f, round(d["value"], 1), round(d["ms_per_step"], 2), d["clocks"]["sm_mhz"], t)
PY
