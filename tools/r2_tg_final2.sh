# tap groups only on <= 128-wide tiles without fused BN: parity, then the bench step A/B/A (3 vs 1)
export CUDA_VISIBLE_DEVICES=0
F=paper_1903_06681_b200/csrc/conv_v2.cu
python -m paper_1903_06681_b200.build > /dev/null
timeout -k 10 900 python -m pytest tests/test_gpu_conv.py tests/test_gpu_edge.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/tgf2_tests.log 2>&1; echo "tests $?"; tail -1 gpurun_out/tgf2_tests.log
cp $F /tmp/conv_v2.g3
for V in 3 1 3; do
  cp /tmp/conv_v2.g3 $F; sed -i "s/^constexpr int kTapGroup = [0-9]*;/constexpr int kTapGroup = $V;/" $F
  python -m paper_1903_06681_b200.build > /dev/null
  timeout -k 10 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/tgf2_$V.json 2> gpurun_out/tgf2_$V.err
  python -c "
import json; d=json.loads(open('gpurun_out/tgf2_$V.json').read().strip().splitlines()[-1])
L=d['config']['layers']; f=lambda n: sum(l['fwd_ms']+l['bwd_ms']+l['bn_stats_ms'] for l in L if l['name'].startswith(n))
print('G=$V', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], 'conv1', round(f('conv1'),2), 'conv2', round(f('conv2'),2), 'conv3', round(f('conv3'),2), 'conv4', round(f('conv4'),2), 'conv5', round(f('conv5'),2), 'conv6', round(f('conv6'),2))"
done
cp /tmp/conv_v2.g3 $F; python -m paper_1903_06681_b200.build > /dev/null
