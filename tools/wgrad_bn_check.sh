# N-tile rule for wgrad_v2: all GPU tests (1 GPU), then the bench
export CUDA_VISIBLE_DEVICES=0
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests8.log 2>&1; echo "tests $?" > gpurun_out/w_status.txt
timeout 600 python bench.py > gpurun_out/bw.json 2> gpurun_out/bw.err; echo "bench $?" >> gpurun_out/w_status.txt
