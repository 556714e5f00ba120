# 2-GPU hang diagnosis: variants of the bench, each bounded
python -m paper_1903_06681_b200.build > /dev/null
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
v() {  # name, extra args
  local n=$1; shift
  NCCL_DEBUG=INFO timeout -k 10 150 $TR --master-port $((29600 + RANDOM % 300)) bench.py --gpus 2 --steps 3 --warmup 3 --watchdog 110 --no-cpu-baseline "$@" > gpurun_out/dbg_$n.out 2> gpurun_out/dbg_$n.err
  echo "$n rc=$? $(python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(d['ms_per_step'])" gpurun_out/dbg_$n.out 2>/dev/null)"
}
v default
v nograph --graph off
v arsync --ar-sync
v arsync_nograph --ar-sync --graph off
v nccl_halo --halo nccl
v mesh1 --workload mesh2k
timeout 900 python -m pytest tests/test_multigpu.py tests/test_redist.py tests/test_cfpar.py -m gpu -x -q --durations=10 > gpurun_out/dbg_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/dbg_tests.log
