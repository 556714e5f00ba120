export CUDA_VISIBLE_DEVICES=0
python -m paper_1903_06681_b200.build > /dev/null
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"bn_bwd" -c 2 -o gpurun_out/ncu_r2_bnsrc python tools/bn_bench.py 8 64 1024 1024 --iters 1 > gpurun_out/ncu_bnsrc.log 2>&1; echo "ncu $?"
