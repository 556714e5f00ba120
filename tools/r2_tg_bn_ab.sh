# same-box A/B/A/B of the bench step: (taps per group 1, fused BN statistics on 128-wide tiles) vs
# (taps per group 3, 128-wide tiles' statistics by the staged pass)
export CUDA_VISIBLE_DEVICES=0
F=paper_1903_06681_b200/csrc/conv_v2.cu; C=paper_1903_06681_b200/csrc/capi.cu
cp $C /tmp/capi.orig
for V in A B A B; do
  cp /tmp/capi.orig $C
  if [ $V = A ]; then G=1; else G=3; sed -i '695s/q.bn <= 128 \&\& (int64_t)q.cin_p \* q.T >= 1152  ? 1/q.bn <= 128 \&\& (int64_t)q.cin_p * q.T >= 1152 \&\& false ? 1/' $C; fi
  sed -i "s/^constexpr int kTapGroup = [0-9]*;/constexpr int kTapGroup = $G;/" $F
  python -m paper_1903_06681_b200.build > /dev/null
  timeout -k 10 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/tgbn_$V.json 2> gpurun_out/tgbn_$V.err
  python -c "
import json; d=json.loads(open('gpurun_out/tgbn_$V.json').read().strip().splitlines()[-1])
L=d['config']['layers']; f=lambda n: sum(l['fwd_ms']+l['bwd_ms']+l['bn_stats_ms'] for l in L if l['name'].startswith(n))
c=[l for l in L if l['name']=='conv2_2'][0]
print('$V', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], 'conv2', round(f('conv2'),2), 'conv3', round(f('conv3'),2), 'conv4', round(f('conv4'),2), 'conv2_2 fwd/bn/bpx/bpw', [round(c[k]*1e3) for k in ('fwd_ms','bn_stats_ms','bwd_data_ms','bwd_filter_ms')])"
done
cp /tmp/capi.orig $C
