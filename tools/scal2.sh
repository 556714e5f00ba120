run() { n=$1; shift; tag=$1; shift; s=$(date +%s); if [ $n = 1 ]; then timeout 400 python bench.py --no-cpu-baseline "$@" > gpurun_out/t_$tag.json 2> gpurun_out/t_$tag.err; else timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2950$n bench.py --gpus $n --no-cpu-baseline "$@" > gpurun_out/t_$tag.json 2> gpurun_out/t_$tag.err; fi; echo "$tag rc=$? $(( $(date +%s)-s ))s" >> gpurun_out/t_times.txt; }
run 2 sp2
run 4 sp4
run 4 sp4_nobn --ablate bn
run 4 sp4_noex --ablate exchange
run 4 sp4_noar --ablate allreduce
run 4 sp4_nobnex --ablate bn,exchange,allreduce
