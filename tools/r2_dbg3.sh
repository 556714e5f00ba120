# 2-GPU: the layer sequence op by op (tools/mg_seq.py), bounded variants
python -m paper_1903_06681_b200.build > /dev/null
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
v() { local n=$1; shift; timeout -k 10 240 $TR --master-port $((29700 + RANDOM % 200)) tools/mg_seq.py "$@" > gpurun_out/seq_$n.log 2>&1; echo "$n rc=$?"; grep -v "^\s*$" gpurun_out/seq_$n.log | grep -v "NCCL INFO\|^W10\|OMP_NUM\|\*\*\*\*" | tail -12; }
v sync_each --sync-each
v plain
v noasync --flags exchange,allreduce,bn
v noexch --flags allreduce,async,bn
v nobn --flags exchange,allreduce,async
v n8 --workload mesh2k_n8
timeout -k 10 300 $TR --master-port 29911 bench.py --gpus 2 --steps 5 --warmup 3 --watchdog 200 --no-cpu-baseline > gpurun_out/seq_bench.json 2> gpurun_out/seq_bench.err; echo "bench rc=$?"; tail -c 300 gpurun_out/seq_bench.json
