# 1-GPU round-2 measurement: smoke, bench lines (bf16, fp32, ResNet-50), the
# GPU suite with durations, the ncu launch list of the default step, full ncu
# captures of the kernels named in the review, the cost-table refit
export CUDA_VISIBLE_DEVICES=0
python -m paper_1903_06681_b200.build > /dev/null
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/p_smoke.log 2>&1; echo "smoke $?"; tail -2 gpurun_out/p_smoke.log
timeout -k 10 600 python bench.py --steps 20 --warmup 5 --watchdog 500 > gpurun_out/p_bench_bf16.json 2> gpurun_out/p_bench_bf16.err; echo "bf16 $?"; tail -c 400 gpurun_out/p_bench_bf16.json
timeout -k 10 900 python bench.py --dtype fp32 --steps 10 --warmup 3 --no-cpu-baseline --watchdog 800 > gpurun_out/p_bench_fp32.json 2> gpurun_out/p_bench_fp32.err; echo "fp32 $?"
timeout -k 10 600 python bench.py --workload resnet50_n64 --steps 20 --warmup 5 --no-cpu-baseline --watchdog 500 > gpurun_out/p_bench_resnet.json 2> gpurun_out/p_bench_resnet.err; echo "resnet $?"
timeout -k 10 600 python bench.py --workload mesh2k_n8_net --steps 10 --warmup 5 --no-cpu-baseline --watchdog 500 > gpurun_out/p_bench_net.json 2> gpurun_out/p_bench_net.err; echo "net $?"
timeout -k 10 2100 python -m pytest tests -m gpu -q --durations=40 > gpurun_out/p_gputests.log 2>&1; echo "gputests $?"; tail -50 gpurun_out/p_gputests.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/p_launches_n8.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/p_ncu_launch.log 2>&1; echo "launches $?"
for spec in "conv1_2_fwd 8 64 1024 1024 64 3 1 1 fwd conv_v2_kernel" "conv3_1_fwd 8 128 512 512 256 3 2 1 fwd conv_v2_kernel" "conv2_1_bpx 8 64 1024 1024 128 3 2 1 bpx conv_v2_kernel" "conv1_1_bpx 8 18 2048 2048 64 3 2 1 bpx conv_v2_kernel"; do
  set -- $spec
  name=$1; shift; sh="$1 $2 $3 $4 $5 $6 $7 $8"; op=$9; k=${10}
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/ncu_r2_$name python tools/kbench.py $sh --ops $op --iters 1 --warmup 1 --flush > gpurun_out/ncu_r2_$name.log 2>&1; echo "ncu $name $?"
done
timeout 1500 python tools/calibrate.py --workloads mesh2k_n8,mesh2k,resnet_layers,resnet50_n64 --out gpurun_out/cost_table_b200_r2.csv > gpurun_out/p_calibrate.log 2>&1; echo "calibrate $?"
