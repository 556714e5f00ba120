# BN backward occupancy A/B on one GPU (the source is edited on the box only)
export CUDA_VISIBLE_DEVICES=0
python -m paper_1903_06681_b200.build > /dev/null
echo "== 1 block/SM, no spills"; for sh in "8 64 1024 1024" "8 256 256 256" "8 512 64 64"; do timeout 120 python tools/bn_bench.py $sh; done
sed -i 's/__launch_bounds__(256, 1) bn_bwd_partials_kernel(/__launch_bounds__(256, 2) bn_bwd_partials_kernel(/; s/__launch_bounds__(256, 1) bn_bwd_apply_kernel(/__launch_bounds__(256, 2) bn_bwd_apply_kernel(/' paper_1903_06681_b200/csrc/bn.cu
python -m paper_1903_06681_b200.build > /dev/null
echo "== 2 blocks/SM, small spills"; for sh in "8 64 1024 1024" "8 256 256 256" "8 512 64 64"; do timeout 120 python tools/bn_bench.py $sh; done
timeout -k 10 600 python -m pytest tests/test_gpu_network.py -m gpu -q > gpurun_out/bnab_tests.log 2>&1; echo "tests $?"; tail -1 gpurun_out/bnab_tests.log
