# HEAD: the ncu launch list of the default bench step (this repo's kernels only; graph off so ncu sees each launch)
export CUDA_VISIBLE_DEVICES=0
python -m paper_1903_06681_b200.build > /dev/null
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"conv_v2|wgrad|bn_|p2p_exchange|redist|cf_|maxpool|import_kernel|weight_|splitk|subpix|subsample|scatter2|block_copy|signal_kernel|conv_gemm|tf32" -c 2000 --csv --log-file gpurun_out/f_launches_n8.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --graph off > gpurun_out/f_ncu.log 2>&1; echo "launches $?"; wc -l gpurun_out/f_launches_n8.csv
