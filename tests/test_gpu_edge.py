"""GPU parity on the degenerate cases of the method (Eq. 1-3, PAPER.md:61-69;
the decomposition of Section IV): 1 x 1 images, outputs of one pixel, single
rows / columns, a filter as large as the image, one channel, and spatial
grids where every rank owns a single row or column -- through the same
checks as tests/test_gpu_conv.py (element-wise derived bounds, north_star
norms, bitwise partition invariance)."""
import pytest
import torch

from tests import test_gpu_conv as tc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dc():
    from paper_1903_06681_b200 import build
    build.build()
    import paper_1903_06681_b200 as dc
    torch.cuda.init()
    return dc


EDGE = [  # (N, C, H, W, F, K, S, P)
    (1, 16, 1, 1, 16, 3, 1, 1),    # 1 x 1 image, every tap but the centre in the padding
    (2, 16, 3, 3, 32, 3, 1, 0),    # valid conv: one output pixel per sample
    (1, 32, 2, 2, 16, 3, 2, 1),    # stride 2 on 2 x 2: one output pixel
    (3, 16, 9, 1, 16, 3, 1, 1),    # one column
    (1, 16, 1, 40, 16, 3, 1, 1),   # one row
    (1, 16, 7, 7, 16, 7, 1, 0),    # filter as large as the image
    (1, 1, 5, 5, 1, 3, 1, 1),      # one channel in, one filter out
    (2, 16, 1, 9, 16, 1, 2, 0),    # 1x1 stride 2 on a single row
]


@pytest.mark.parametrize("shape", EDGE)
def test_edge_single_gpu(dc, shape):
    tc.test_single_gpu_parity(dc, shape)


@pytest.mark.parametrize("shape,grid", [
    ((1, 16, 4, 4, 16, 3, 1, 1), (1, 4, 1)),   # one owned row per rank
    ((1, 16, 4, 4, 16, 3, 1, 1), (1, 1, 4)),   # one owned column per rank
    ((2, 16, 3, 3, 16, 3, 1, 1), (1, 3, 1)),
    ((4, 16, 2, 2, 16, 3, 1, 1), (4, 1, 1)),   # one sample per rank
])
def test_edge_partition_bitwise(dc, shape, grid):
    tc.test_partition_bitwise(dc, shape, grid)


@pytest.mark.parametrize("case", [
    ((1, 16, 1, 1, 32, 3, 1, 1), (1, 1, 1)),   # one pixel per channel: variance 0, y_hat 0
    ((2, 16, 1, 1, 48, 3, 1, 1), (1, 1, 1)),   # two pixels per channel
])
def test_edge_bn_one_gpu(dc, case):
    """BN apply / backward (reading R27) on the smallest statistics groups."""
    from tests import test_gpu_network as tn
    tn.test_bn_apply_backward_one_gpu(dc, case, True, True)
    tn.test_bn_apply_backward_one_gpu(dc, case, False, False)


@pytest.mark.parametrize("shape,grid", [
    ((1, 16, 1, 1, 3, 1, 1), (1, 1, 1)),    # 1 x 1 image: the window is the pixel itself
    ((2, 16, 3, 3, 3, 2, 0), (1, 1, 1)),    # one output pixel
    ((1, 16, 5, 5, 1, 1, 0), (1, 1, 1)),    # K = 1: identity
    ((2, 16, 8, 4, 3, 2, 1), (1, 4, 1)),    # two input rows per rank, windows across two ranks
])
def test_edge_maxpool(dc, shape, grid):
    """Max pooling with its halo exchange (reading R31)
    on the smallest windows and shards."""
    from tests import test_pool as tp
    tp.test_maxpool_parity(dc, shape, grid)
