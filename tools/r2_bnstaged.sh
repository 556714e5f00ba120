# Staged (bulk-copy) BN kernels on one GPU: parity, microbench, network step, ncu of the backward
export CUDA_VISIBLE_DEVICES=0
python -m paper_1903_06681_b200.build > /dev/null
timeout -k 10 900 python -m pytest tests/test_gpu_network.py tests/test_pool.py -m gpu -q -x > gpurun_out/bnst_tests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/bnst_tests.log
for sh in "8 64 1024 1024" "8 256 256 256" "8 512 64 64" "8 64 512 512"; do timeout 120 python tools/bn_bench.py $sh; done
timeout -k 10 600 python bench.py --workload mesh2k_n8_net --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bnst_net.json 2> gpurun_out/bnst_net.err; echo "net $?"; cat gpurun_out/bnst_net.json
timeout -k 10 300 ncu --set full --clock-control none -k regex:bn_staged -c 3 -o gpurun_out/bnst_ncu python tools/bn_bench.py 8 64 1024 1024 --iters 1 > gpurun_out/bnst_ncu.log 2>&1; echo "ncu $?"
