# conv2_x pipeline A/B (source edited on the box only): CTA-pair multicast of weight stages, A stage depth
export CUDA_VISIBLE_DEVICES=0
L="8 128 512 512 128 3 1 1"; L3="8 256 256 256 256 3 1 1"
run() { python -m paper_1903_06681_b200.build > /dev/null; for s in "$L" "$L3"; do timeout 120 python tools/kbench.py $s --ops fwd,bpx --flush --iters 10; done; }
echo "== HEAD"; run
cp paper_1903_06681_b200/csrc/conv_v2.cu /tmp/conv_v2.cu.orig
sed -i 's/    p.cluster = (!p.b_resident \&\& p.bn % 32 == 0 \&\& p.kind == 0) ? 2 : 1;/    p.cluster = 1;/' paper_1903_06681_b200/csrc/conv_v2.cu
echo "== no CTA-pair multicast"; run
cp /tmp/conv_v2.cu.orig paper_1903_06681_b200/csrc/conv_v2.cu
sed -i 's/^        p.a_stages = 2;$/        p.a_stages = 3;/' paper_1903_06681_b200/csrc/conv_v2.cu
echo "== 3 A stages"; run
cp /tmp/conv_v2.cu.orig paper_1903_06681_b200/csrc/conv_v2.cu
