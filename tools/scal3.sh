run() { n=$1; shift; tag=$1; shift; s=$(date +%s); timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2950$n bench.py --gpus $n --no-cpu-baseline "$@" > gpurun_out/u_$tag.json 2> gpurun_out/u_$tag.err; echo "$tag rc=$? $(( $(date +%s)-s ))s" >> gpurun_out/u_times.txt; }
run 4 h4 --decomp 1,4,1
DC_NO_OVERLAP=1 run 4 h4_noov --decomp 1,4,1
DC_FUSED_HALO=1 run 4 h4_fused --decomp 1,4,1
DC_NO_OVERLAP=1 run 4 sp4_noov
DC_FUSED_HALO=1 run 4 sp4_fused
run 4 w4 --decomp 1,1,4
