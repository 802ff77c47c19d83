"""K3 tree/causal/full attention over the paged KV cache vs a dense torch fp32 reference."""

import math

import pytest
import torch

pytestmark = pytest.mark.gpu


def _setup(n_q, n_kv, c, s, seed, n_layers=2, layer=1):
    from paper_2605_29727_b200.engine.forward import PagedKV
    g = torch.Generator(device="cuda").manual_seed(seed)
    kv = PagedKV(n_layers, n_kv, c + s + 64, "cuda")
    # scramble the page table to exercise paging
    perm = torch.randperm(kv.n_pages, generator=torch.Generator().manual_seed(seed)).to(torch.int32).cuda()
    kv.page_table.copy_(perm)
    kv.buf.normal_(0, 1, generator=g)
    q = torch.randn(s, n_q * 128, device="cuda", generator=g).to(torch.bfloat16)
    return kv, q


def _gather(kv, layer, n_kv, slots, which):
    """[len(slots), n_kv, 128] fp32 from the paged cache."""
    L = kv.buf.view(kv.n_layers, kv.n_pages, 2, n_kv, 64, 128)
    pages = kv.page_table[slots // 64].long()
    off = slots % 64
    return L[layer, pages, which, :, off].float()  # [n, n_kv, 128]


def pack_mask(bits, words):
    import numpy as np
    pad = np.zeros((bits.shape[0], words * 32), dtype=bool)
    pad[:, : bits.shape[1]] = bits
    return np.packbits(pad, axis=1, bitorder="little").view(np.uint32).view(np.int32).copy()


def _ref(q, kv, layer, n_q, n_kv, c, s, visible):
    keys = torch.arange(c + s, device="cuda")
    K = _gather(kv, layer, n_kv, keys, 0)
    V = _gather(kv, layer, n_kv, keys, 1)
    g = n_q // n_kv
    K = K.repeat_interleave(g, 1)
    V = V.repeat_interleave(g, 1)
    qf = q.float().view(s, n_q, 128)
    sc = torch.einsum("qhd,khd->hqk", qf, K) / math.sqrt(128)
    sc = sc.masked_fill(~visible[None], float("-inf"))
    return torch.einsum("hqk,khd->qhd", torch.softmax(sc, -1), V).reshape(s, n_q * 128)


@pytest.fixture(params=["tc", "kt"])
def variant(request):
    """K3 entry point under test: bst_attention (shape-selected row-major tcgen05 kernels)
    or bst_attention_keymajor."""
    return request.param == "kt"


@pytest.mark.parametrize("n_q,n_kv", [(32, 8), (4, 2)])
@pytest.mark.parametrize("c,s", [(0, 1), (5, 17), (2048, 17), (300, 65), (1000, 256), (4096, 33), (20000, 17), (9000, 100),
                                 (300, 600), (2048, 1025)])
@pytest.mark.parametrize("splits", [0, 1])
def test_tree_attention(n_q, n_kv, c, s, splits, variant):
    from oracle import specplan_port as O
    from paper_2605_29727_b200 import ops
    kv, q = _setup(n_q, n_kv, c, s, seed=c + s)
    # random tree over s rows (parent[i] < i)
    gen = torch.Generator().manual_seed(s)
    parent = [-1] + [int(torch.randint(0, i, (1,), generator=gen)) for i in range(1, s)]
    import numpy as np
    anc = torch.from_numpy(O.ancestor_bits(np.array(parent))).cuda()
    words = (s + 31) // 32
    packed = torch.from_numpy(pack_mask(anc.cpu().numpy(), words)).cuda()
    out = torch.empty(s, n_q * 128, device="cuda", dtype=torch.bfloat16)
    ws = torch.zeros(8 << 20, device="cuda", dtype=torch.float32)
    ops.attention(q, out, kv.buf, 2, kv.n_pages, 1, kv.page_table, n_q, n_kv, s, c, s, c + s, None, 0, packed.view(-1),
                  words, ws, n_splits=splits, keymajor=variant)
    vis = torch.zeros(s, c + s, dtype=torch.bool, device="cuda")
    vis[:, :c] = True
    vis[:, c:] = anc
    ref = _ref(q, kv, 1, n_q, n_kv, c, s, vis)
    torch.cuda.synchronize()
    err = (out.float() - ref).abs().max().item()
    assert err < 2e-2, err


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("c,s", [(0, 64), (130, 40), (1900, 17)])
def test_causal_and_full_attention_with_device_c(mode, c, s, variant):
    from paper_2605_29727_b200 import ops
    n_q, n_kv = 32, 8
    kv, q = _setup(n_q, n_kv, c, s, seed=7 + c)
    state = torch.tensor([c, 0, 0, 0, 0, 0, 0, 0], dtype=torch.int32, device="cuda")
    out = torch.empty(s, n_q * 128, device="cuda", dtype=torch.bfloat16)
    ws = torch.zeros(8 << 20, device="cuda", dtype=torch.float32)
    ops.attention(q, out, kv.buf, 2, kv.n_pages, 1, kv.page_table, n_q, n_kv, s, 0, s, c + s + 64, state, mode,
                  None, 0, ws, keymajor=variant)
    vis = torch.zeros(s, c + s, dtype=torch.bool, device="cuda")
    vis[:, :c] = True
    if mode == 1:
        vis[:, c:] = torch.tril(torch.ones(s, s, dtype=torch.bool, device="cuda"))
    else:
        vis[:, c:] = True
    ref = _ref(q, kv, 1, n_q, n_kv, c, s, vis)
    torch.cuda.synchronize()
    assert (out.float() - ref).abs().max().item() < 2e-2


@pytest.mark.parametrize("c", [2048, 20000])
def test_back_to_back_launches_in_a_graph(c, variant):
    """PDL lets the CTAs of the next K3 launch start while the previous one merges its
    splits; the alternating workspace banks keep them apart (layer parity).  A graph of
    back-to-back launches over distinct layers must reproduce the eager results bitwise."""
    from paper_2605_29727_b200 import ops
    from paper_2605_29727_b200.engine.forward import PagedKV
    n_q, n_kv, s, L = 32, 8, 17, 6
    g = torch.Generator(device="cuda").manual_seed(c)
    kv = PagedKV(L, n_kv, c + s + 64, "cuda")
    kv.buf.normal_(0, 1, generator=g)
    q = torch.randn(s, n_q * 128, device="cuda", generator=g).to(torch.bfloat16)
    words = 1
    anc = torch.full((s, words), -1, dtype=torch.int32, device="cuda")
    ws = torch.zeros(8 << 20, device="cuda", dtype=torch.float32)
    outs = [torch.empty(s, n_q * 128, device="cuda", dtype=torch.bfloat16) for _ in range(L)]

    def run():
        for li in range(L):
            ops.attention(q, outs[li], kv.buf, L, kv.n_pages, li, kv.page_table, n_q, n_kv, s, c, s, c + s, None, 0,
                          anc.view(-1), words, ws, keymajor=variant)
    run()
    torch.cuda.synchronize()
    want = [o.clone() for o in outs]
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        run()
    st.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=st):
        run()
    for _ in range(3):
        for o in outs:
            o.zero_()
        torch.cuda.synchronize()
        with torch.cuda.stream(st):
            graph.replay()
        st.synchronize()
        for o, w in zip(outs, want):
            assert torch.equal(o, w)


@pytest.mark.parametrize("c,s", [(2048, 96), (2048, 17)])
def test_cluster_merge_large_values(c, s):
    """The cluster split merge stages each split's normalised rows as fp16 (a convex
    combination of V rows): V rows ~1e3 (far above LLM value activations, below fp16's
    65504) still match the dense fp32 reference to bf16 precision."""
    from oracle import specplan_port as O
    from paper_2605_29727_b200 import ops
    import numpy as np
    n_q, n_kv = 32, 8
    kv, q = _setup(n_q, n_kv, c, s, seed=c + 3 * s)
    L = kv.buf.view(kv.n_layers, kv.n_pages, 2, n_kv, 64, 128)
    L[:, :, 1].mul_(1000.0)  # V pages only
    gen = torch.Generator().manual_seed(s)
    parent = [-1] + [int(torch.randint(0, i, (1,), generator=gen)) for i in range(1, s)]
    anc = torch.from_numpy(O.ancestor_bits(np.array(parent))).cuda()
    words = (s + 31) // 32
    packed = torch.from_numpy(pack_mask(anc.cpu().numpy(), words)).cuda()
    out = torch.empty(s, n_q * 128, device="cuda", dtype=torch.bfloat16)
    ws = torch.zeros(8 << 20, device="cuda", dtype=torch.float32)
    ops.attention(q, out, kv.buf, 2, kv.n_pages, 1, kv.page_table, n_q, n_kv, s, c, s, c + s, None, 0, packed.view(-1),
                  words, ws)
    vis = torch.zeros(s, c + s, dtype=torch.bool, device="cuda")
    vis[:, :c] = True
    vis[:, c:] = anc
    ref = _ref(q, kv, 1, n_q, n_kv, c, s, vis)
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    err = (out.float() - ref).abs().max().item()
    assert err < 2e-2 * 1000.0, err
