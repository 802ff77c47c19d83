"""K4 tcgen05 GEMM vs a torch fp32 reference of the same bf16 operands."""

import pytest
import torch

pytestmark = pytest.mark.gpu

SHAPES = [(64, 64, 5), (200, 136, 1), (6144, 4096, 17), (4096, 4096, 1), (24576, 4096, 33), (4096, 12288, 100),
          (1024, 4096, 256), (300, 4096, 256), (4096, 20480, 17), (151936, 4096, 17), (128, 64, 16),
          # pair mode (two weight tiles per stream-K unit, bn > 128), odd tile counts included
          (24576, 4096, 256), (151936, 4096, 144), (37888, 4096, 200), (18944, 512, 256)]


@pytest.mark.parametrize("n_out,k,m", SHAPES)
def test_gemm_matches_fp32_reference(n_out, k, m):
    from paper_2605_29727_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(n_out + k + m)
    x = torch.randn(m, k, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(n_out, k, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    y = ops.linear(x, w)
    ref = x.float() @ w.float().t()
    torch.cuda.synchronize()
    err = (y - ref).abs().max().item()
    scale = ref.abs().max().item()
    assert err <= 1e-4 * scale + 1e-5, (err, scale)


def test_gemm_strided_x_and_determinism():
    from paper_2605_29727_b200 import ops
    x_full = torch.randn(40, 4096 + 64, device="cuda").to(torch.bfloat16)
    x = x_full[:, :4096]
    w = (torch.randn(4096, 4096, device="cuda") * 0.02).to(torch.bfloat16)
    y1 = ops.linear(x, w)
    y2 = ops.linear(x, w)
    assert torch.equal(y1, y2)
    ref = x.float() @ w.float().t()
    assert (y1 - ref).abs().max().item() < 1e-3


def test_gemm_argmax_lowest_index_ties():
    from paper_2605_29727_b200 import ops
    k, n_out, m = 256, 5000, 9
    x = torch.zeros(m, k, device="cuda", dtype=torch.bfloat16)
    x[:, 0] = 1.0
    w = torch.zeros(n_out, k, device="cuda", dtype=torch.bfloat16)
    w[[17, 400, 4999], 0] = 2.0  # three-way tie -> 17
    w[3000, 0] = 1.5
    am = ops.gemm_argmax(ops.gemm_partial(x, w))
    assert am.tolist() == [17] * m
    x2 = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    w2 = (torch.randn(n_out, k, device="cuda") * 0.05).to(torch.bfloat16)
    am2 = ops.gemm_argmax(ops.gemm_partial(x2, w2))
    ref = (x2.float() @ w2.float().t()).argmax(dim=1).int()
    assert torch.equal(am2, ref)


@pytest.mark.parametrize("n_out,k,m", [(24576, 4096, 256), (4096, 12288, 160), (1024, 4096, 136), (256, 200, 129),
                                       (200, 4096, 250), (4096, 4096, 512), (24576, 4096, 455), (6144, 4096, 300)])
def test_cta_pair_gemm_matches_single_cta_kernel(n_out, k, m):
    """The CTA-pair kernel (tcgen05 cta_group::2, schedule cta2) against the one-CTA
    kernel on the same operands: fp32 partials reduce to the same Y up to summation order,
    and repeated launches are bitwise identical."""
    from paper_2605_29727_b200 import ops
    s = ops.gemm_schedule(n_out, k, m, 148)
    assert s.cta2 == 1 and s.pair == 2 and s.grid == min(74, s.units)
    g = torch.Generator(device="cuda").manual_seed(m)
    x = torch.randn(m, k, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(n_out, k, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    y1 = ops.linear(x, w)
    y2 = ops.linear(x, w)
    assert torch.equal(y1, y2)
    # the same product through the one-CTA kernel: split X into <= 128-row chunks
    ref = torch.cat([ops.linear(x[i:i + 128], w) for i in range(0, m, 128)])
    exact = x.float() @ w.float().t()
    scale = exact.abs().max().item()
    assert (y1 - exact).abs().max().item() <= 1e-4 * scale + 1e-5
    assert (y1 - ref).abs().max().item() <= 1e-4 * scale + 1e-5
