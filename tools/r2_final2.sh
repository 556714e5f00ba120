# final 2-GPU check at HEAD: the multi-GPU tests, then the bench at N = 1, 2
export NCCL_DEBUG=WARN
python -m paper_1903_06681_b200.build > /dev/null
timeout -k 10 900 python -m pytest tests/test_multigpu.py tests/test_multigpu_fullsize.py tests/test_redist.py tests/test_cfpar.py -m gpu -q > gpurun_out/f2_tests.log 2>&1; echo "tests $?"; tail -2 gpurun_out/f2_tests.log
timeout -k 10 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29952 bench.py --gpus 2 --steps 20 --warmup 5 --watchdog 500 > gpurun_out/f2_bench2.json 2> gpurun_out/f2_bench2.err; echo "n2 $?"
timeout -k 10 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29953 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/f2_ref2.json 2> gpurun_out/f2_ref2.err; echo "ref n2 $?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/f2_bench2.json").read().strip().splitlines()[-1])
print(2, round(d["value"], 1), round(d["ms_per_step"], 2), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
print(open("gpurun_out/f2_ref2.json").read().strip()[:200])
PY
