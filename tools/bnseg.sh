# fused BN statistics for layers with several N tiles (per-CTA segments): parity, then bench A/B
export CUDA_VISIBLE_DEVICES=0
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests7.log 2>&1; echo "tests $?" > gpurun_out/g_status.txt
timeout 600 python bench.py > gpurun_out/bg_new.json 2> gpurun_out/bg_new.err; echo "bench $?" >> gpurun_out/g_status.txt
DC_BN_FUSE_NT1=1 timeout 600 python bench.py > gpurun_out/bg_old.json 2> gpurun_out/bg_old.err; echo "bench_old $?" >> gpurun_out/g_status.txt
timeout 600 python bench.py > gpurun_out/bg_new2.json 2> gpurun_out/bg_new2.err; echo "bench2 $?" >> gpurun_out/g_status.txt
