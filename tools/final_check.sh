# final round-1 confirmation of the default path: all GPU tests, smoke, bench, launch list
export CUDA_VISIBLE_DEVICES=0
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_final.log 2>&1; echo "tests $?" > gpurun_out/final_status.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_final.log 2>&1; echo "smoke $?" >> gpurun_out/final_status.txt
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench $?" >> gpurun_out/final_status.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'conv_v2|wgrad|bn_|splitk|weight_transform|subpix' -c 4000 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_final.log 2>&1; echo "L $?" >> gpurun_out/final_status.txt
