# streamed-weight MMA loop issuing taps in pairs: parity, layer times, the bench step
export CUDA_VISIBLE_DEVICES=0
python -m paper_1903_06681_b200.build > /dev/null
timeout -k 10 900 python -m pytest tests/test_gpu_conv.py tests/test_gpu_edge.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/tp_tests.log 2>&1; echo "tests $?"; tail -2 gpurun_out/tp_tests.log
for s in "8 128 512 512 128 3 1 1" "8 256 256 256 256 3 1 1" "8 512 128 128 512 3 1 1" "8 128 512 512 256 3 2 1" "8 512 64 64 512 3 1 1"; do timeout 60 python tools/kbench.py $s --ops fwd,bpx --flush --iters 10 2>&1 | tail -2; done
timeout -k 10 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/tp_bench.json 2> gpurun_out/tp_bench.err; echo "bench $?"
