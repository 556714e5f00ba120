# Staged BN statistics: parity (conv BN tests, network, multi-rank loopback), then the bench step
export CUDA_VISIBLE_DEVICES=0
python -m paper_1903_06681_b200.build > /dev/null
timeout -k 10 900 python -m pytest tests/test_gpu_conv.py tests/test_gpu_network.py tests/test_pool.py tests/test_loopback.py -m gpu -q -x -k "bn or BN or stats or network or pool or loopback" > gpurun_out/bnstats_tests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/bnstats_tests.log
timeout -k 10 600 python bench.py --steps 10 --warmup 5 > gpurun_out/bnstats_bench.json 2> gpurun_out/bnstats_bench.err; echo "bench $?"
timeout -k 10 600 python bench.py --workload mesh2k_n8_net --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bnstats_net.json 2> gpurun_out/bnstats_net.err; echo "net $?"
for sh in "8 256 256 256" "8 64 1024 1024"; do timeout 120 python tools/bn_bench.py $sh --iters 50; done
