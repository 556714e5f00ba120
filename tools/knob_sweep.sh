# knob sweep on the slowest-per-FLOP ops of the mesh2k_n8 step (kbench, cold L2)
export CUDA_VISIBLE_DEVICES=0
K="timeout 120 python tools/kbench.py"
o=gpurun_out/knobs.txt
run() { echo "== $1 :: $2" >> $o; env $1 $K $2 --flush --iters 20 --warmup 5 >> $o 2>&1; }
for e in "X=0" "DC_WGRAD_BW8=1" "DC_WGRAD_SM_GBS=25" "DC_WGRAD_SM_GBS=80" "DC_WGRAD_BN=256"; do
  run "$e" "8 512 128 128 512 3 1 1 --ops bpw"
  run "$e" "8 64 1024 1024 64 3 1 1 --ops bpw"
  run "$e" "8 256 256 256 256 3 1 1 --ops bpw"
done
for e in "X=0" "DC_SERIAL_PHASES=1"; do
  run "$e" "8 64 1024 1024 128 3 2 1 --ops bpx"
  run "$e" "8 128 512 512 256 3 2 1 --ops bpx"
done
for e in "X=0" "DC_V2_BN=128"; do
  run "$e" "8 512 128 128 512 3 1 1 --ops fwd,bpx --bn-fused"
  run "$e" "8 256 256 256 256 3 1 1 --ops fwd,bpx --bn-fused"
done
echo done >> $o
