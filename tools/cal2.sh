timeout 600 python tools/calibrate.py --workloads mesh2k_n8 --out gpurun_out/ct_n8b.csv > gpurun_out/cal2.log 2>&1
python tools/merge_tables.py profiles/cost_table_b200.csv gpurun_out/ct_n8b.csv; cp profiles/cost_table_b200.csv gpurun_out/ct_merged2.csv
timeout 600 python bench.py > gpurun_out/b1n8b.json 2> gpurun_out/b1n8b.err; echo "bench $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:dc:: -c 4000 --csv --log-file gpurun_out/launches_n8.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "L $?"
