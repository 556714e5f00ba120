export CUDA_VISIBLE_DEVICES=0
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -x --durations=0 > gpurun_out/fullsize.log 2>&1; echo "full $?" > gpurun_out/fz_status.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_f.log 2>&1; echo "smoke $?" >> gpurun_out/fz_status.txt
