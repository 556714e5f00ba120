# streamed-weight MMA loop: taps per wait group 1 / 2 / 3 / 4 (source edited on the box), then parity at the default
export CUDA_VISIBLE_DEVICES=0
F=paper_1903_06681_b200/csrc/conv_v2.cu
cp $F /tmp/conv_v2.orig
run() { python -m paper_1903_06681_b200.build > /dev/null; for s in "8 128 512 512 128 3 1 1" "8 256 256 256 256 3 1 1" "8 512 128 128 512 3 1 1" "8 128 512 512 256 3 2 1" "8 512 64 64 512 3 1 1"; do timeout 60 python tools/kbench.py $s --ops fwd,bpx --flush --iters 10 2>&1 | tail -2; done; }
for G in 1 2 4 3; do
  sed -i "s/^constexpr int kTapGroup = [0-9]*;/constexpr int kTapGroup = $G;/" $F
  echo "== taps per group $G"; run
done
timeout -k 10 900 python -m pytest tests/test_gpu_conv.py tests/test_gpu_edge.py tests/test_gpu_fullsize.py tests/test_loopback.py -m gpu -q -x > gpurun_out/tg_tests.log 2>&1; echo "tests $?"; tail -2 gpurun_out/tg_tests.log
timeout -k 10 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/tg_bench.json 2> gpurun_out/tg_bench.err; echo "bench $?"
