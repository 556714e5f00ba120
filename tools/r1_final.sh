# round-1 final GPU pass: parity tests, bench, launch list, conv1_1 forward capture
export CUDA_VISIBLE_DEVICES=0
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests3.log 2>&1; echo "tests $?" > gpurun_out/f_status.txt
timeout 600 python bench.py > gpurun_out/bf.json 2> gpurun_out/bf.err; echo "bench $?" >> gpurun_out/f_status.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'conv_v2|wgrad|bn_|splitk|weight_transform|subpix' -c 4000 --csv --log-file gpurun_out/launches_f.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_f.log 2>&1; echo "L $?" >> gpurun_out/f_status.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:conv_v2_kernel -c 1 -o gpurun_out/ncu_fwd_conv1_1_n8 python tools/kbench.py 8 18 2048 2048 64 3 2 1 --ops fwd --bn-fused --iters 1 --warmup 1 > gpurun_out/ncu_f11.log 2>&1; echo "f11 $?" >> gpurun_out/f_status.txt
