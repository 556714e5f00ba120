# same-box A/B of the bench step: taps per wait group 1 vs 3 (ABAB)
export CUDA_VISIBLE_DEVICES=0
F=paper_1903_06681_b200/csrc/conv_v2.cu
for G in 1 3 1 3; do
  sed -i "s/^constexpr int kTapGroup = [0-9]*;/constexpr int kTapGroup = $G;/" $F
  python -m paper_1903_06681_b200.build > /dev/null
  timeout -k 10 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/tgb_$G.json 2> gpurun_out/tgb_$G.err
  python -c "
import json; d=json.loads(open('gpurun_out/tgb_$G.json').read().strip().splitlines()[-1])
L=d['config']['layers']; f=lambda n: sum(l['fwd_ms']+l['bwd_ms'] for l in L if l['name'].startswith(n))
print('G=$G', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], 'conv2', round(f('conv2'),2), 'conv3', round(f('conv3'),2), 'conv4', round(f('conv4'),2), 'conv5', round(f('conv5'),2))"
done
