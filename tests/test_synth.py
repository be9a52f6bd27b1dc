"""The seeded input generators: determinism and the structural contract of the CSR."""
import numpy as np

from synth import get_config, make_graph, make_inputs, make_block_parts, small_config
from synth.configs import scaled


def _check_csr(ip, ix, n):
    assert ip[0] == 0 and ip[-1] == ix.size and ip.dtype == np.int64 and ix.dtype == np.int32
    rows = np.repeat(np.arange(n), np.diff(ip))
    assert np.all(ix != rows)                                   # no self loops
    key = rows * n + ix
    assert np.all(np.diff(key) > 0)                             # sorted, no duplicates
    rev = np.sort(ix.astype(np.int64) * n + rows)
    assert np.array_equal(rev, key)                             # symmetric


def test_cora_shape_and_determinism():
    cfg = get_config("cora")
    ip, ix = make_graph(cfg)
    assert ix.size == cfg.nnz
    _check_csr(ip, ix, cfg.num_nodes)
    ip2, ix2 = make_graph(cfg)
    assert np.array_equal(ip, ip2) and np.array_equal(ix, ix2)


def test_inputs_padding_and_parts():
    cfg = get_config("cora")
    inp = make_inputs(cfg)
    assert inp.x.shape == (cfg.num_nodes, 1436) and np.all(inp.x[:, 1433:] == 0)
    assert inp.weights[0].shape == (1436, 16) and np.all(inp.weights[0][1433:] == 0)
    assert inp.weights[1].shape == (16, 8) and np.all(inp.weights[1][:, 7:] == 0)
    assert int(inp.train_mask.sum()) == 140
    for M in (1, 2, 4, 8):
        p = make_block_parts(cfg, M)
        assert np.bincount(p, minlength=M).min() > 0 and np.all(np.diff(p) >= 0)


def test_scaled_and_small():
    for name in ("flickr", "arxiv", "reddit", "products"):
        c = scaled(get_config(name), 0.002)
        ip, ix = make_graph(c)
        assert ix.size == c.nnz
        _check_csr(ip, ix, c.num_nodes)
    c = small_config()
    ip, ix = make_graph(c)
    _check_csr(ip, ix, c.num_nodes)
