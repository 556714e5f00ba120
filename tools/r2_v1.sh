# 1-GPU verification at HEAD: GPU suite, smoke, bench lines, BN microbenchmark
export CUDA_VISIBLE_DEVICES=0
python -m paper_1903_06681_b200.build > /dev/null
timeout -k 10 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/v_gputests.log 2>&1; echo "gputests $?"; tail -22 gpurun_out/v_gputests.log
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; echo "smoke $?"; tail -1 gpurun_out/v_smoke.log
for sh in "8 64 1024 1024" "8 256 256 256" "8 512 64 64"; do timeout 120 python tools/bn_bench.py $sh; done
for wl in mesh2k_n8 resnet50_n64 mesh2k_n8_net; do
  timeout -k 10 600 python bench.py --workload $wl --steps 20 --warmup 5 --watchdog 500 $( [ $wl != mesh2k_n8 ] && echo --no-cpu-baseline ) > gpurun_out/v_bench_$wl.json 2> gpurun_out/v_bench_$wl.err; echo "$wl $?"
done
python - <<'PY'
import json
for wl in ("mesh2k_n8", "resnet50_n64", "mesh2k_n8_net"):
    try:
        d = json.loads(open(f"gpurun_out/v_bench_{wl}.json").read().strip().splitlines()[-1])
    except Exception as e:
        print(wl, "no result", e); continue
    t = {}
    for l in d["config"]["layers"]:
        for k, v in l.items():
            if k.endswith("_ms") and k != "model_pred_ms":
                t[k] = round(t.get(k, 0) + v, 2)
    print(wl, round(d["value"], 1), round(d["ms_per_step"], 2), d["clocks"]["sm_mhz"], round(d["roofline"]["frac"], 3), t)
PY
