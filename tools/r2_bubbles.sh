# DIAGNOSTIC (results wrong on purpose, timing only): which wait starves the conv2_x MMA stream
export CUDA_VISIBLE_DEVICES=0
F=paper_1903_06681_b200/csrc/conv_v2.cu
cp $F /tmp/conv_v2.orig
L="8 128 512 512 128 3 1 1"; L1="8 64 1024 1024 64 3 1 1"
run() { python -m paper_1903_06681_b200.build > /dev/null; for s in "$L" "$L1"; do timeout 60 python tools/kbench.py $s --ops fwd --flush --iters 10 2>&1 | tail -1; done; }
echo "== HEAD"; run
sed -i '616s|st_global_v8(orow + c16 \* 16, pk);|if (p.nout_p < 0) st_global_v8(orow + c16 * 16, pk);|' $F
echo "== no epilogue stores"; run
cp /tmp/conv_v2.orig $F
sed -i '412s|mbar_wait(&b_full\[sb\], ph);|if (p.nout_p < 0) mbar_wait(\&b_full[sb], ph);|' $F
echo "== MMA does not wait for weight stages"; run
cp /tmp/conv_v2.orig $F
sed -i '380s|mbar_wait(&a_full\[s\], (a_it / p.a_stages) \& 1);|if (p.nout_p < 0) mbar_wait(\&a_full[s], (a_it / p.a_stages) \& 1);|' $F
echo "== MMA does not wait for input stages"; run
cp /tmp/conv_v2.orig $F
python -m paper_1903_06681_b200.build > /dev/null
