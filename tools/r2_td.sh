export NCCL_DEBUG=WARN
python -m paper_1903_06681_b200.build > /dev/null
timeout -k 10 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29961 bench.py --gpus 2 --steps 10 --warmup 5 --watchdog 300 > gpurun_out/t_bench2.json 2> gpurun_out/t_bench2.err; echo "n2 rc=$?"; tail -c 200 gpurun_out/t_bench2.json; grep -A3 Timeout gpurun_out/t_bench2.err | head
timeout -k 10 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29962 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/t_ref2.json 2> gpurun_out/t_ref2.err; echo "ref2 rc=$?"; tail -c 200 gpurun_out/t_ref2.json
