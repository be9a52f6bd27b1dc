"""Pins for the bf16 stale store option of the oracle: the rounding
routine against the library definition and hand-computed ties, and the store semantics."""
import numpy as np
import torch

from oracle import oracle_train
from oracle.train import bf16_round
from synth import small_config, make_inputs, make_random_parts


def test_bf16_round_matches_torch_and_ties():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(20000) * 10.0 ** rng.integers(-6, 6, 20000),
                        [0.0, -0.0, 1.0, -2.5, 3.0e38, 1e-40]])
    ref = torch.from_numpy(x.astype(np.float32)).to(torch.bfloat16).to(torch.float64).numpy()
    np.testing.assert_array_equal(bf16_round(x), ref)
    # ties to even at 1.0 (bf16 spacing 2^-7): 1+2^-8 -> 1, 1+3*2^-8 -> 1+2^-6
    assert bf16_round(1 + 2.0 ** -8) == 1.0
    assert bf16_round(1 + 3 * 2.0 ** -8) == 1 + 2.0 ** -6
    assert bf16_round(-(1 + 2.0 ** -8 + 2.0 ** -20)) == -(1 + 2.0 ** -7)
    # relative error bound of round-to-nearest with 8 significant bits
    y = rng.uniform(-4, 4, 10000)
    assert (np.abs(bf16_round(y) - y) <= np.abs(y) * 2.0 ** -8 * (1 + 1e-6)).all()


def _inp(seed):
    cfg = small_config(num_nodes=44, nnz=200, d0=5, hidden=(6, 5), num_classes=3, c_pad=4,
                       seed=seed, train_frac=0.6)
    return cfg, make_inputs(cfg)


def test_bf16_store_is_exact_without_halo():
    cfg, inp = _inp(3)
    part = np.zeros(cfg.num_nodes, np.int32)
    kw = dict(sync_interval=1, epochs=3, lr=0.3)
    a = oracle_train(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                     cfg.num_classes, part, 1, store_dtype="bf16", **kw)
    b = oracle_train(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                     cfg.num_classes, part, 1, **kw)
    for wa, wb in zip(a.weights, b.weights):
        np.testing.assert_array_equal(wa, wb)


def test_bf16_store_pulls_rounded_rows():
    """lr = 0, N = 1: the halo used at epoch 2 is the bf16 rounding of epoch 1's
    representations of those nodes (SPEC S:377 with the rounding applied)."""
    cfg, inp = _inp(5)
    M = 3
    part = make_random_parts(cfg.num_nodes, M, 2)
    run = oracle_train(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                       cfg.num_classes, part, M, sync_interval=1, epochs=2, lr=0.0,
                       record_outputs=True, store_dtype="bf16")
    r1, r2 = run.records
    for l in (1, 2):
        for m, p in enumerate(run.parts):
            np.testing.assert_array_equal(r2.halo_used[(l, m)], bf16_round(r1.reps[l][p.halo_ids]))
            assert not np.array_equal(r2.halo_used[(l, m)], r1.reps[l][p.halo_ids])
