"""CPU check of the row-window identities tests/test_gpu_fullsize.py uses to
compute sampled full-size outputs with the oracle: Eq. 1 / Eq. 3 on a row
window (same padding) equals the full oracle's row, exactly, for every row
(halo slicing; strides and P < O, P = O, P > S)."""
import numpy as np
import pytest

import datagen
import oracle
from tests.test_gpu_fullsize import _bwd_window, _fwd_window


@pytest.mark.parametrize("shape", [(2, 3, 17, 9, 4, 3, 2, 1), (1, 2, 16, 8, 3, 3, 1, 1), (1, 2, 11, 7, 2, 1, 1, 0),
                                   (1, 2, 20, 9, 2, 5, 2, 2), (1, 2, 13, 9, 2, 3, 2, 0), (1, 2, 12, 8, 2, 5, 1, 1),
                                   (1, 3, 30, 14, 4, 7, 2, 3), (1, 2, 25, 9, 2, 7, 1, 3)])
def test_row_windows_equal_full_oracle(shape):
    N, C, H, W, F, K, S, P = shape
    x, w = datagen.gen_x(N, C, H, W), datagen.gen_w(F, C, K)
    Ho, Wo = oracle.out_extent(H, K, S, P), oracle.out_extent(W, K, S, P)
    dy = datagen.gen_dy(N, F, Ho, Wo)
    y, dx = oracle.conv_fwd(x, w, S, P), oracle.conv_bwd_data(dy, w, H, W, S, P)
    for n in range(N):
        for i in range(Ho):
            r0, L, ip = _fwd_window(i, H, K, S, P)
            ref = oracle.conv_fwd(x[n:n + 1, :, r0:r0 + L], w, S, P, rows=(ip, ip + 1))[0, :, ip, :]
            assert np.array_equal(ref, y[n, :, i, :])
        for u in range(H):
            i0, i1, Hl, up = _bwd_window(u, Ho, H, K, S, P)
            ref = oracle.conv_bwd_data(dy[n:n + 1, :, i0:i1], w, Hl, W, S, P, rows=(up, up + 1))[0, :, up, :]
            assert np.array_equal(ref, dx[n, :, u, :])
