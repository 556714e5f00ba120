for sh in "8 18 2048 2048 64 3 2 1" "8 64 1024 1024 64 3 1 1" "8 64 1024 1024 128 3 2 1" "8 128 512 512 128 3 1 1" "8 128 512 512 256 3 2 1" "8 256 256 256 256 3 1 1" "8 256 256 256 512 3 2 1" "8 512 128 128 512 3 1 1" "8 512 128 128 512 3 2 1" "8 512 64 64 512 3 1 1" "8 512 32 32 512 3 1 1" "8 64 256 1024 64 3 1 1" "8 128 64 512 256 3 2 1" "8 512 16 64 512 3 1 1"; do
  for v in 200 55 40; do
    r=$(DC_WGRAD_SM_GBS=$v timeout 120 python tools/kbench.py $sh --ops bpw --iters 10 --flush 2>&1 | tail -1)
    echo "$sh gbs=$v : $r" >> gpurun_out/wsplit.txt
  done
done
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/gputests2.log 2>&1; echo "tests $?" >> gpurun_out/wsplit.txt
