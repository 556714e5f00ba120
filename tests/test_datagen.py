"""The torch (device) form of the counter-based input generator must produce
exactly the numpy generator's values (DESIGN.md §3 input recipe): the bench
builds its resident inputs with it on the GPU."""
import numpy as np
import pytest
import torch

import datagen


@pytest.mark.parametrize("kind", ["act", "act24", "weight"])
def test_datagen_torch_matches_numpy(kind):
    shape = (3, 18, 37, 29)
    blk = dict(n=(1, 3), c=(2, 17), h=(5, 30), w=(3, 29))
    a = datagen.gen_block(shape, 1903, 2, kind, scale=0.25, **blk)
    b = datagen.gen_block_nhwc_torch(shape, 1903, 2, kind, scale=0.25, c_pad=24, **blk)
    assert b.shape == (2, 25, 26, 24)
    assert np.array_equal(a.transpose(0, 2, 3, 1), b[..., :15].numpy())
    assert torch.count_nonzero(b[..., 15:]) == 0


def test_datagen_torch_bf16_exact():
    """act values are bf16-exact, so the bf16 tensor holds the same numbers."""
    a = datagen.gen_x(1, 8, 16, 16)
    b = datagen.gen_block_nhwc_torch((1, 8, 16, 16), datagen.SEED, datagen.TID_X, dtype=torch.bfloat16)
    assert np.array_equal(a.transpose(0, 2, 3, 1), b.double().numpy())
