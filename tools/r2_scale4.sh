# one 4-GPU box: the GPU suite's multi-GPU tests, then the bench at N = 1, 2, 4 back to back (the driver's scaling run)
export NCCL_DEBUG=WARN
python -m paper_1903_06681_b200.build > /dev/null
timeout -k 10 900 python -m pytest tests/test_multigpu.py tests/test_multigpu_fullsize.py tests/test_redist.py tests/test_cfpar.py -m gpu -q > gpurun_out/s_tests.log 2>&1; echo "tests $?"; tail -2 gpurun_out/s_tests.log
CUDA_VISIBLE_DEVICES=0 timeout -k 10 600 python bench.py --steps 20 --warmup 5 --watchdog 500 > gpurun_out/s_bench1.json 2> gpurun_out/s_bench1.err; echo "n1 $?"
for n in 2 4; do
  timeout -k 10 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2995$n bench.py --gpus $n --steps 20 --warmup 5 --watchdog 500 > gpurun_out/s_bench$n.json 2> gpurun_out/s_bench$n.err; echo "n$n $?"
done
python - <<'PY'
import json
base = None
for n in (1, 2, 4):
    try:
        d = json.loads(open(f"gpurun_out/s_bench{n}.json").read().strip().splitlines()[-1])
    except Exception as e:
        print(n, "no result", e); continue
    base = base or d["value"]
    print(n, round(d["value"], 1), round(d["ms_per_step"], 2), "eff", round(d["value"] / (n * base), 3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
