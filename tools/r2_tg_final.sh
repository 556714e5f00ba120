# tap groups (3, not with fused BN statistics): parity + the bench step (A/B against tap group 1)
export CUDA_VISIBLE_DEVICES=0
F=paper_1903_06681_b200/csrc/conv_v2.cu
python -m paper_1903_06681_b200.build > /dev/null
timeout -k 10 900 python -m pytest tests/test_gpu_conv.py tests/test_gpu_edge.py tests/test_gpu_fullsize.py tests/test_loopback.py tests/test_gpu_network.py -m gpu -q -x > gpurun_out/tgf_tests.log 2>&1; echo "tests $?"; tail -2 gpurun_out/tgf_tests.log
cp $F /tmp/conv_v2.g3
for V in 3 1 3; do
  cp /tmp/conv_v2.g3 $F; sed -i "s/^constexpr int kTapGroup = [0-9]*;/constexpr int kTapGroup = $V;/" $F
  python -m paper_1903_06681_b200.build > /dev/null
  timeout -k 10 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/tgf_$V.json 2> gpurun_out/tgf_$V.err
  python -c "
import json; d=json.loads(open('gpurun_out/tgf_$V.json').read().strip().splitlines()[-1])
L=d['config']['layers']; f=lambda n: sum(l['fwd_ms']+l['bwd_ms']+l['bn_stats_ms'] for l in L if l['name'].startswith(n))
c=[l for l in L if l['name']=='conv2_2'][0]
print('G=$V', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], 'conv2', round(f('conv2'),2), 'conv3', round(f('conv3'),2), 'conv4', round(f('conv4'),2), 'conv5', round(f('conv5'),2), 'conv2_2', [round(c[k]*1e3) for k in ('fwd_ms','bn_stats_ms','bwd_data_ms','bwd_filter_ms')])"
done
cp /tmp/conv_v2.g3 $F; python -m paper_1903_06681_b200.build > /dev/null
