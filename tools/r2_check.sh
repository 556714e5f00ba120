# 2-GPU check: GPU suite (1- and 2-GPU tests), redistribution tests, 2-GPU bench teardown
export NCCL_DEBUG=WARN
python -m paper_1903_06681_b200.build > /dev/null
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2c_gputests.log 2>&1; echo "gputests rc=$?"; tail -3 gpurun_out/r2c_gputests.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 --steps 10 --warmup 5 > gpurun_out/r2c_bench2.json 2> gpurun_out/r2c_bench2.err; echo "bench2 rc=$?"; tail -c 600 gpurun_out/r2c_bench2.json; grep -A30 "Thread\|Stack\|Timeout" gpurun_out/r2c_bench2.err | head -60
