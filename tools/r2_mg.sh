# multi-GPU round-2 measurement on P GPUs (P = number visible): bench, halo /
# redistribution / channel-parallel microbenchmarks, new multi-GPU tests,
# C5 sweep + E7, ResNet-50 sample vs hybrid, network-level strategy
P=$(nvidia-smi -L | wc -l)
export NCCL_DEBUG=WARN
python -m paper_1903_06681_b200.build > /dev/null
run() {  # name, timeout, command...
  local n=$1 t=$2; shift 2
  timeout -k 20 $t "$@" > gpurun_out/mg${P}_$n.out 2> gpurun_out/mg${P}_$n.err; echo "$n rc=$?"
}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1"
run bench 420 $TR --master-port 29532 bench.py --gpus $P --steps 10 --warmup 5 --watchdog 300
tail -c 300 gpurun_out/mg${P}_bench.out; grep -A12 "Thread 0x\|most recent call first" gpurun_out/mg${P}_bench.err | head -40
run halo 300 $TR --master-port 29530 tools/halo_bench.py; cat gpurun_out/mg${P}_halo.out
run redist 600 $TR --master-port 29531 tools/redist_bench.py; cat gpurun_out/mg${P}_redist.out
run tests 1500 python -m pytest tests/test_cfpar.py tests/test_redist.py tests/test_multigpu.py -m gpu -x -q --durations=15; tail -25 gpurun_out/mg${P}_tests.out
for dec in strategy spatial; do
  run net_$dec 420 $TR --master-port 29535 bench.py --gpus $P --workload mesh2k_n8_net --decomp $dec --steps 10 --warmup 5 --watchdog 300
  python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['config'].get('strategy',{}).get('model_step_ms'))" gpurun_out/mg${P}_net_$dec.out
done
for dec in "$P,1,1" "$((P/2)),2,1"; do
  run resnet_${dec//,/_} 420 $TR --master-port 29534 bench.py --gpus $P --workload resnet50_n64 --decomp $dec --steps 10 --warmup 5 --watchdog 300
  python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'])" gpurun_out/mg${P}_resnet_${dec//,/_}.out
done
# halo hiding: the same step with the non-overlapped schedule and with the exchanges removed (diagnostic)
run noov 420 $TR --master-port 29536 bench.py --gpus $P --steps 10 --warmup 5 --no-overlap --watchdog 300
python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print('no-overlap',d['value'],d['ms_per_step'])" gpurun_out/mg${P}_noov.out
run noex 420 $TR --master-port 29537 bench.py --gpus $P --steps 10 --warmup 5 --ablate exchange --watchdog 300
python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print('no-exchange',d['value'],d['ms_per_step'])" gpurun_out/mg${P}_noex.out
run c5 1500 $TR --master-port 29533 tools/c5_sweep.py --out gpurun_out/c5_e7_${P}gpu.jsonl; tail -25 gpurun_out/mg${P}_c5.out
