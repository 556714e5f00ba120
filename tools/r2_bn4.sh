export CUDA_VISIBLE_DEVICES=0
python -m paper_1903_06681_b200.build > /dev/null
timeout -k 10 900 python -m pytest tests/test_gpu_network.py tests/test_pool.py tests/test_gpu_fp32.py -m gpu -q > gpurun_out/e_tests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/e_tests.log
for sh in "8 64 1024 1024" "8 256 256 256" "8 512 64 64"; do timeout 120 python tools/bn_bench.py $sh; done
timeout 300 ncu --set full --clock-control none -k regex:"bn_bwd" -c 2 -o gpurun_out/ncu_r2_bnb2 python tools/bn_bench.py 8 64 1024 1024 --iters 1 > gpurun_out/ncu_bnb2.log 2>&1; echo "ncu $?"
