# DIAGNOSTIC (results wrong on purpose, timing only): is the conv2_x streamed-weight kernel bound by the MMAs?
export CUDA_VISIBLE_DEVICES=0
F=paper_1903_06681_b200/csrc/conv_v2.cu
cp $F /tmp/conv_v2.orig
L="8 128 512 512 128 3 1 1"; L3="8 256 256 256 256 3 1 1"
run() { python -m paper_1903_06681_b200.build > /dev/null; for s in "$L" "$L3"; do timeout 60 python tools/kbench.py $s --ops fwd --flush --iters 10 2>&1 | tail -1; done; }
echo "== HEAD"; run
sed -i '419s|issue_slot_any<KIND>(nk16, p.tpw, d_tmem, ad, bd,|issue_slot_any<KIND>(nk16, 1, d_tmem, ad, bd,|' $F
echo "== half the MMAs (second tile of each pair skipped)"; run
cp /tmp/conv_v2.orig $F
sed -i '414s|const uint64_t ad = arow + (uint32_t)(tw >> p.s_shift) \* p.a_col16 +|const uint64_t ad = a_stage + 0 * (arow + (uint32_t)(tw >> p.s_shift) * p.a_col16) +|' $F
echo "== every tap reads the unshifted A window"; run
cp /tmp/conv_v2.orig $F
python -m paper_1903_06681_b200.build > /dev/null
