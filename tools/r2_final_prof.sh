# HEAD evidence: the ncu launch list of the default bench step, ncu --set full of the staged BN kernels
export CUDA_VISIBLE_DEVICES=0
python -m paper_1903_06681_b200.build > /dev/null
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/f_launches_n8.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/f_ncu_launch.log 2>&1; echo "launches $?"
timeout 400 ncu --set full --clock-control none --import-source on -k regex:bn_staged -s 3 -c 3 -o gpurun_out/f_bn_staged python tools/bn_bench.py 8 64 1024 1024 --iters 1 > gpurun_out/f_bn_ncu.log 2>&1; echo "ncu bn $?"
