# ncu --set full of conv2_2 forward (C = F = 128) and conv1_2 forward (64), one launch each
export CUDA_VISIBLE_DEVICES=0
python -m paper_1903_06681_b200.build > /dev/null
timeout 120 python tools/kbench.py 8 128 512 512 128 3 1 1 --ops fwd --flush --iters 10
timeout 300 ncu --set full --import-source on --clock-control none -k regex:conv_v2 -s 1 -c 1 -o gpurun_out/conv2_2_fwd python tools/kbench.py 8 128 512 512 128 3 1 1 --ops fwd --iters 1 --warmup 1 > gpurun_out/conv2prof.log 2>&1; echo "ncu $?"
