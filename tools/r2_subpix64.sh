# stride-2 backward-data with 64 input channels: four phase GEMMs (HEAD) vs the sub-pixel GEMM (N = 4 x 64)
export CUDA_VISIBLE_DEVICES=0
run() { python -m paper_1903_06681_b200.build > /dev/null; for s in "8 64 1024 1024 128 3 2 1" "8 64 256 256 128 3 2 1" "8 32 1024 1024 64 3 2 1"; do timeout 120 python tools/kbench.py $s --ops bpx --flush --iters 10; done; }
echo "== phases (HEAD)"; run
sed -i 's/if (g.dt != 0 || g.S != 2 || g.Cp > 32 || pl->scat_seg) return false;/if (g.dt != 0 || g.S != 2 || g.Cp > 64 || pl->scat_seg) return false;/' paper_1903_06681_b200/csrc/capi.cu
echo "== sub-pixel up to 64 channels"; run
timeout -k 10 600 python -m pytest tests/test_gpu_conv.py tests/test_gpu_edge.py -m gpu -q -x 2>&1 | tail -2
