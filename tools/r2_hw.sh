# 2 or 4 GPUs: the in-kernel halo wait -- multi-GPU parity tests, then the bench with and without it
export NCCL_DEBUG=WARN
P=$(nvidia-smi -L | wc -l)
python -m paper_1903_06681_b200.build > /dev/null
timeout -k 10 900 python -m pytest tests/test_multigpu.py tests/test_redist.py -m gpu -q -x > gpurun_out/h_tests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/h_tests.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1"
for v in default noov; do
  extra=""; [ $v = noov ] && extra="--no-overlap"
  timeout -k 10 400 $TR --master-port $((29970 + RANDOM % 20)) bench.py --gpus $P --steps 20 --warmup 5 --watchdog 300 $extra > gpurun_out/h_bench_$v.json 2> gpurun_out/h_bench_$v.err; echo "$v rc=$?"
  python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[1], d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])" gpurun_out/h_bench_$v.json
done
