# BN statistics pass A/B on one GPU: the staged kernel (working tree) vs bn_sums_kernel (HEAD, built in a copy)
export CUDA_VISIBLE_DEVICES=0
python -m paper_1903_06681_b200.build > /dev/null
echo "== staged"; for sh in "8 256 256 256" "8 128 512 512" "8 512 128 128" "8 512 32 32"; do timeout 120 python tools/bn_bench.py $sh --iters 50 | grep stats; done
rm -rf /tmp/old && mkdir /tmp/old && cp -r . /tmp/old/ 2>/dev/null; cd /tmp/old && cp tools/old_halo.cu paper_1903_06681_b200/csrc/halo.cu && cp tools/old_halo.cuh paper_1903_06681_b200/csrc/halo.cuh && cp tools/old_capi.cu paper_1903_06681_b200/csrc/capi.cu && python -m paper_1903_06681_b200.build > /dev/null
echo "== bn_sums_kernel"; for sh in "8 256 256 256" "8 128 512 512" "8 512 128 128" "8 512 32 32"; do timeout 120 python tools/bn_bench.py $sh --iters 50 | grep stats; done
