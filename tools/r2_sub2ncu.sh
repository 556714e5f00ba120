export CUDA_VISIBLE_DEVICES=0
python -m paper_1903_06681_b200.build > /dev/null
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sub2_launches.csv python tools/kbench.py 64 1024 14 14 2048 1 2 0 --iters 1 --warmup 1 > /dev/null 2>&1; echo "ncu $?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r50b2b_launches.csv python tools/kbench.py 64 512 7 7 512 3 1 1 --iters 1 --warmup 1 > /dev/null 2>&1; echo "ncu $?"
