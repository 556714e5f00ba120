# A/B of the second epilogue warp group (DC_V2_EPI4=1 turns it off)
export CUDA_VISIBLE_DEVICES=0
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests4.log 2>&1; echo "tests $?" > gpurun_out/e_status.txt
for sh in "8 18 2048 2048 64 3 2 1" "8 64 1024 1024 64 3 1 1" "8 64 1024 1024 128 3 2 1" "8 128 512 512 128 3 1 1" "8 256 256 256 256 3 1 1" "8 512 128 128 512 3 1 1" "8 512 32 32 512 3 1 1"; do
  for e in 0 1; do
    if [ $e = 1 ]; then export DC_V2_EPI4=1; else unset DC_V2_EPI4; fi
    echo "== $sh epi4=$e" >> gpurun_out/epi_ab.txt
    timeout 120 python tools/kbench.py $sh --ops fwd,bpx --bn-fused --flush --iters 20 --warmup 5 >> gpurun_out/epi_ab.txt 2>&1
  done
done
unset DC_V2_EPI4
echo "ab done" >> gpurun_out/e_status.txt
timeout 600 python bench.py > gpurun_out/be.json 2> gpurun_out/be.err; echo "bench $?" >> gpurun_out/e_status.txt
