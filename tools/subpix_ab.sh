# A/B: sub-pixel backward-data for 64-channel stride-2 layers (DC_SUBPIX_MAXC=64)
export CUDA_VISIBLE_DEVICES=0
DC_SUBPIX_MAXC=64 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests6.log 2>&1; echo "tests64 $?" > gpurun_out/s_status.txt
for sh in "8 64 1024 1024 128 3 2 1" "1 64 1024 1024 128 3 2 1" "8 32 1024 1024 64 3 2 1"; do
  for m in 32 64; do
    echo "== $sh maxc=$m" >> gpurun_out/subpix_ab.txt
    DC_SUBPIX_MAXC=$m timeout 120 python tools/kbench.py $sh --ops bpx --flush --iters 20 --warmup 5 >> gpurun_out/subpix_ab.txt 2>&1
  done
done
timeout 600 python bench.py > gpurun_out/bs1.json 2> gpurun_out/bs1.err; echo "bench $?" >> gpurun_out/s_status.txt
DC_SUBPIX_MAXC=64 timeout 600 python bench.py > gpurun_out/bs64.json 2> gpurun_out/bs64.err; echo "bench64 $?" >> gpurun_out/s_status.txt
