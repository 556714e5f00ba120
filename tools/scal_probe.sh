set -x
run() { n=$1; shift; tag=$1; shift; s=$(date +%s); if [ $n = 1 ]; then timeout 400 python bench.py --no-cpu-baseline "$@" > gpurun_out/s_$tag.json 2> gpurun_out/s_$tag.err; else timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2950$n bench.py --gpus $n --no-cpu-baseline "$@" > gpurun_out/s_$tag.json 2> gpurun_out/s_$tag.err; fi; echo "$tag rc=$? $(( $(date +%s)-s ))s" >> gpurun_out/s_times.txt; }
run 1 n8_1 --workload mesh2k_n8
run 2 n8_2 --workload mesh2k_n8
run 4 n8_4 --workload mesh2k_n8
run 2 n8_2s --workload mesh2k_n8 --decomp 1,2,1
run 4 n8_4s --workload mesh2k_n8 --decomp 1,4,1
run 4 n1_4 --workload mesh2k
