# wgrad_v2 N-tile width 128 vs 256 across local work sizes (kbench, cold L2)
export CUDA_VISIBLE_DEVICES=0
o=gpurun_out/wgrad_bn.txt
for sh in "512 128 128 512" "256 256 256 256" "512 64 64 512" "512 32 32 512" "256 128 128 512"; do
  set -- $sh
  for n in 1 2 4 8; do
    for bn in 128 256; do
      echo "== N=$n C=$1 H=$2 W=$3 F=$4 bn=$bn" >> $o
      if [ "$1" = "256" ] && [ "$4" = "512" ]; then args="$n $1 $2 $3 $4 3 2 1"; h=$2; else args="$n $1 $2 $3 $4 3 1 1"; fi
      DC_WGRAD_BN=$bn timeout 120 python tools/kbench.py $args --ops bpw --flush --iters 20 --warmup 5 >> $o 2>&1
    done
  done
done
echo done >> $o
