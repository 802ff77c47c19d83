"""Shared helpers of the engine GPU tests (not a test module)."""

import numpy as np
import torch

from oracle import specplan_port as O


def _prompt(n, V, seed=0):
    return np.random.default_rng(seed).integers(0, V - 1, n).tolist()


def _replay_check(eng, exported, tokens, policy, dims=None, t_draft=0.0, t_aux=0.0, l_ar=1.0, n_max=64):
    """Run the ORACLE decode loop on the GPU-exported fp64 rows + verify argmax: must be bit-identical."""
    P = eng.prompt_len
    by_prefix = {}
    committed = []
    for e in exported:
        by_prefix[tuple(committed)] = e
        committed = committed + [int(e["token"][i]) for i in e["path"][1:]] + [e["bonus"]]

    def drafter(prefix):
        return by_prefix[tuple(prefix)]["probs"]

    def target(seq, T):
        for k in range(len(seq), -1, -1):  # find the cycle whose prefix this seq extends
            e = by_prefix.get(tuple(seq[:k]))
            if e is None:
                continue
            walk = seq[k:]
            node = 0
            kids = {}
            for i in range(1, len(e["parent"])):
                kids.setdefault(int(e["parent"][i]), {})[int(e["token"][i])] = i
            for t in walk:
                node = kids[node][t]
            return int(e["argmax"][node])
        raise KeyError(seq)

    run_len = len(tokens)
    records, toks = O.decode_loop(drafter, target, run_len, eng.top_k, policy, n_max, dims, P - 1, t_draft, t_aux,
                                  l_ar)
    assert list(toks) == list(tokens)
    for rec, e in zip(records, exported):
        assert rec["tree_size"] == int(e["meta"][0])
        assert rec["surrogate"] == e["surrogate"]
    return records


def _decoy_drafter(ar, gamma, V, seed):
    """Test drafter: the target's greedy token competes with decoys so the accepted path is non-contiguous."""
    rng = np.random.default_rng(seed)

    def fn(e):
        k = int(e.state[3].item())  # committed so far
        lg = torch.zeros(gamma, V, device="cuda")
        for j in range(gamma):
            dec = int(rng.integers(0, V))
            lg[j, dec] = 10.3  # a decoy ranked above the target's token
            if k + j < len(ar):
                lg[j, ar[k + j]] = 10.0
        return lg
    return fn
