# A/B of CTA pairs on resident-weight 64/128-channel layers (DC_V2_CG2R=1), cold L2
for e in "" "DC_V2_CG2R=1"; do
  echo "#### env: $e"
  env $e timeout 120 python tools/kbench.py 8 64 1024 1024 64 3 1 1 --flush --ops fwd,bpx --bn-fused --iters 10
  env $e timeout 120 python tools/kbench.py 8 128 512 512 128 3 1 1 --flush --ops fwd,bpx --bn-fused --iters 10
  env $e timeout 120 python tools/kbench.py 32 64 56 56 64 3 1 1 --flush --ops fwd,bpx --iters 10
done
DC_V2_CG2R=1 timeout 600 python -m pytest tests/test_gpu_conv.py -q -x -k "single_gpu_parity or partition_bitwise or fused_bn" 2>&1 | tail -3
