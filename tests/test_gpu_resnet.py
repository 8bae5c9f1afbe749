"""GPU parity on every distinct ResNet-50 conv shape (proj/data/resnet_layers.csv,
BASELINE.json configs[2]): 7x7/s2 stem, 1x1 s1/s2 bottlenecks, 3x3 -- at a
reduced batch so the oracle finishes in seconds.  TF32 / BF16 tensor-core
paths within the stated tolerances; the exact FP32 path bit-identical."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

# (name, window, stride, in HxWxC, out HxWxK)
RESNET = [
    ("conv1", 7, 2, (224, 224, 3), (112, 112, 64)),
    ("res2a_branch2a", 1, 1, (56, 56, 64), (56, 56, 64)),
    ("res2a_branch2b", 3, 1, (56, 56, 64), (56, 56, 64)),
    ("res2a_branch2c", 1, 1, (56, 56, 64), (56, 56, 256)),
    ("res2a_branch1", 1, 1, (56, 56, 64), (56, 56, 256)),
    ("res2b_branch2a", 1, 1, (56, 56, 256), (56, 56, 64)),
    ("res3a_branch2a", 1, 2, (56, 56, 256), (28, 28, 128)),
    ("res3a_branch2b", 3, 1, (28, 28, 128), (28, 28, 128)),
    ("res3a_branch2c", 1, 1, (28, 28, 128), (28, 28, 512)),
    ("res3a_branch1", 1, 2, (56, 56, 256), (28, 28, 512)),
    ("res3b_branch2a", 1, 1, (28, 28, 512), (28, 28, 128)),
    ("res4a_branch2a", 1, 2, (28, 28, 512), (14, 14, 256)),
    ("res4a_branch2b", 3, 1, (14, 14, 256), (14, 14, 256)),
    ("res4a_branch2c", 1, 1, (14, 14, 256), (14, 14, 1024)),
    ("res4a_branch1", 1, 2, (28, 28, 512), (14, 14, 1024)),
    ("res4b_branch2a", 1, 1, (14, 14, 1024), (14, 14, 256)),
    ("res5a_branch2a", 1, 2, (14, 14, 1024), (7, 7, 512)),
    ("res5a_branch2b", 3, 1, (7, 7, 512), (7, 7, 512)),
    ("res5a_branch2c", 1, 1, (7, 7, 512), (7, 7, 2048)),
    ("res5a_branch1", 1, 2, (14, 14, 1024), (7, 7, 2048)),
    ("res5b_branch2a", 1, 1, (7, 7, 2048), (7, 7, 512)),
]
TOL = {"tf32": 1e-3, "bf16": 5e-3}


def case(tk, oracle, row, batch):
    name, r, stride, (h, w, c), (oh, ow, k) = row
    same = oh == (h + stride - 1) // stride  # layers.hpp:37-40
    s = tk.ConvShape(batch, h, w, c, k, r, r, stride, same)
    conv = oracle.Conv(batch, h, w, c, k, r, r, stride, same)
    assert (conv.out_rows, conv.out_cols) == (oh, ow)
    x = oracle.fill_random(int(np.prod(conv.in_shape)), 11).reshape(conv.in_shape)
    f = oracle.fill_random(int(np.prod(conv.filt_shape)), 12).reshape(conv.filt_shape)
    return s, conv, x, f


@pytest.mark.parametrize("row", RESNET, ids=[r[0] for r in RESNET])
@pytest.mark.parametrize("prec", ["tf32", "bf16"])
def test_resnet_layer_tensor_cores(tk, oracle, row, prec):
    import torch
    s, conv, x, f = case(tk, oracle, row, 2)
    want = oracle.conv2d_naive(conv, x, f)
    dx, df = torch.from_numpy(x).cuda(), torch.from_numpy(f).cuda()
    dy = torch.full(conv.out_shape, float("nan"), device="cuda")
    tk.conv2d_dev(dx, df, dy, s, tk.parse_conv_params("im2col"), precision=prec)
    torch.cuda.synchronize()
    got = dy.cpu().numpy()
    assert not np.isnan(got).any()
    assert oracle.max_scaled_error(got, want) <= TOL[prec]


@pytest.mark.parametrize("row", RESNET[::4], ids=[r[0] for r in RESNET[::4]])
def test_resnet_layer_exact(tk, oracle, row):
    s, conv, x, f = case(tk, oracle, row, 1)
    want = oracle.conv2d_naive(conv, x, f)
    got = tk.conv2d(x, f, s, tk.parse_conv_params("tiled_t4x4_v4x4"))
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.timeout(120)
def test_gather_mode_many_tiles_many_slabs(tk, oracle):
    """Regression: res3a_branch2a (1x1/s2, C=256) at batch 32 runs the gather
    producer with several tiles per CTA and more K-slabs per tile than
    pipeline stages (the configuration that once deadlocked).  Images 0 and
    31 are checked against single-image oracle runs."""
    import torch
    N, H, C, K = 32, 56, 256, 128
    s = tk.ConvShape(N, H, H, C, K, 1, 1, 2, True)
    gen = torch.Generator(device="cuda").manual_seed(3)
    dx = torch.rand((N, H, H, C), device="cuda", generator=gen) * 2 - 1
    df = torch.rand((1, 1, C, K), device="cuda", generator=gen) * 2 - 1
    dy = torch.empty(s.out_shape, device="cuda")
    # 1x1 layers default to the pointwise GEMM: force the gather producers
    tk.conv2d_dev(dx, df, dy, s, tk.parse_conv_params("im2col"),
                  options=tk.exec_options("tf32", mode="gather"))
    torch.cuda.synchronize()
    f = df.cpu().numpy()
    for img in (0, N - 1):
        conv = oracle.Conv(1, H, H, C, K, 1, 1, 2, True)
        want = oracle.conv2d_naive(conv, dx[img:img + 1].cpu().numpy(), f)
        assert oracle.max_scaled_error(dy[img:img + 1].cpu().numpy(), want) <= TOL["tf32"]


@pytest.mark.timeout(120)
@pytest.mark.parametrize("prec", ["tf32", "bf16"])
@pytest.mark.parametrize("row", [RESNET[20], RESNET[19], RESNET[15], RESNET[13]],
                         ids=["res5b_branch2a", "res5a_branch1", "res4b_branch2a",
                              "res4a_branch2c"])
def test_pointwise_full_batch_split_k(tk, oracle, row, prec):
    """1x1 layers at batch 32 run as a plain GEMM on the NHWC input, split
    over K with a deterministic reduction where the output has few tiles:
    images 0 and 31 against the oracle, and two runs bit-identical."""
    import torch
    name, r, stride, (h, w, c), (oh, ow, k) = row
    N = 32
    s = tk.ConvShape(N, h, w, c, k, 1, 1, stride, True)
    gen = torch.Generator(device="cuda").manual_seed(5)
    dx = torch.rand((N, h, w, c), device="cuda", generator=gen) * 2 - 1
    df = torch.rand((1, 1, c, k), device="cuda", generator=gen) * 2 - 1
    ys = []
    for _ in range(2):
        dy = torch.full(s.out_shape, float("nan"), device="cuda")
        tk.conv2d_dev(dx, df, dy, s, tk.parse_conv_params("im2col"), precision=prec)
        ys.append(dy)
    torch.cuda.synchronize()
    assert torch.equal(ys[0].view(torch.int32), ys[1].view(torch.int32))
    f = df.cpu().numpy()
    for img in (0, N - 1):
        conv = oracle.Conv(1, h, w, c, k, 1, 1, stride, True)
        want = oracle.conv2d_naive(conv, dx[img:img + 1].cpu().numpy(), f)
        assert oracle.max_scaled_error(ys[0][img:img + 1].cpu().numpy(), want) <= TOL[prec]
