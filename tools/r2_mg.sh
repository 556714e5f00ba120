# multi-GPU round-2 measurement on P GPUs (P = number visible): new multi-GPU
# tests, C5 sweep + E7, redistribution / channel-parallel microbenchmarks, bench
P=$(nvidia-smi -L | wc -l)
export NCCL_DEBUG=WARN
python -m paper_1903_06681_b200.build > /dev/null
timeout 1200 python -m pytest tests/test_cfpar.py tests/test_redist.py tests/test_multigpu.py -m gpu -x -q > gpurun_out/mg${P}_newtests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/mg${P}_newtests.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 29530 tools/halo_bench.py > gpurun_out/halo_bench_${P}gpu.jsonl 2> gpurun_out/halo_bench_${P}gpu.err; echo "halo rc=$?"; cat gpurun_out/halo_bench_${P}gpu.jsonl
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 29531 tools/redist_bench.py --out gpurun_out/redist_bench_${P}gpu.jsonl > gpurun_out/redist_bench_${P}gpu.log 2>&1; echo "redist rc=$?"; cat gpurun_out/redist_bench_${P}gpu.jsonl
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus $P --steps 10 --warmup 5 > gpurun_out/mg${P}_bench.json 2> gpurun_out/mg${P}_bench.err; echo "bench rc=$?"; tail -c 400 gpurun_out/mg${P}_bench.json
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 29533 tools/c5_sweep.py --out gpurun_out/c5_e7_${P}gpu.jsonl > gpurun_out/c5_${P}gpu.log 2>&1; echo "c5 rc=$?"; tail -25 gpurun_out/c5_${P}gpu.log
# ResNet-50 conv stack (configs[1]/[2], C2): sample vs hybrid grids
for dec in "$P,1,1" "$((P/2)),2,1"; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus $P --workload resnet50_n64 --decomp $dec --steps 10 --warmup 5 > gpurun_out/mg${P}_resnet_${dec//,/_}.json 2> gpurun_out/mg${P}_resnet_${dec//,/_}.err; echo "resnet $dec rc=$?"; python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'])" gpurun_out/mg${P}_resnet_${dec//,/_}.json
done
# network level (E7): the model's strategy (per-layer grids + shuffles) and its pure-spatial restriction
for dec in strategy spatial; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus $P --workload mesh2k_n8_net --decomp $dec --steps 10 --warmup 5 > gpurun_out/mg${P}_net_${dec}.json 2> gpurun_out/mg${P}_net_${dec}.err; echo "net $dec rc=$?"; python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['config'].get('strategy',{}).get('model_step_ms'))" gpurun_out/mg${P}_net_${dec}.json
done
