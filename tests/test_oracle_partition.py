"""Pins for oracle O1-O6 (propagation values and the partition split)."""
import numpy as np
import pytest

from oracle import oracle_partition, prop_values, degrees
from tests.brute import brute_partition, dense_P
from tests.helpers import csr_from_edges, golden, random_graph, random_parts

G = golden("spec_examples.json")


def _dense_from_part(p, n_nodes):
    """Expand P_in + P_out back to global columns (S:116 reconstruction)."""
    gid = np.concatenate([p.local_ids, p.halo_ids]).astype(np.int64)
    out = np.zeros((p.n_local, n_nodes))
    for i in range(p.n_local):
        for e in range(p.row_ptr[i], p.row_ptr[i + 1]):
            out[i, gid[p.col[e]]] += p.val[e]
    return out


def test_prop_worked_examples():
    for key in ("prop_two_nodes", "prop_isolated"):
        ex = G[key]
        ip, ix = csr_from_edges(ex["n"], ex["edges"])
        p = oracle_partition(ip, ix, np.zeros(ex["n"], np.int32), 1, 0)
        np.testing.assert_array_equal(_dense_from_part(p, ex["n"]), np.array(ex["P"]))
    ex = G["prop_path"]
    ip, ix = csr_from_edges(3, ex["edges"])
    d = _dense_from_part(oracle_partition(ip, ix, np.zeros(3, np.int32), 1, 0), 3)
    assert abs(d[1, 1] - ex["P11"]) < 1e-7 and abs(d[0, 1] - ex["P01"]) < 1e-7


def test_prop_bits():
    for dv, du, bits in G["prop_bits"]["pairs"]:
        got = prop_values(np.array([dv]), np.array([du])).view(np.uint32)[0]
        assert got == int(bits, 16), (dv, du, hex(got))


def test_prop_symmetric_and_regular_rows():
    # 4-regular circulant on 11 nodes: every row of P sums to 1
    n = 11
    edges = [(v, (v + s) % n) for v in range(n) for s in (1, 2)]
    ip, ix = csr_from_edges(n, edges)
    d = _dense_from_part(oracle_partition(ip, ix, np.zeros(n, np.int32), 1, 0), n)
    np.testing.assert_array_equal(d, d.T)
    np.testing.assert_allclose(d.sum(1), 1.0, atol=1e-6)


def test_value_formula_matches_dense_definition():
    """The pinned rounding A2 equals fp32 of the fp64 matrix definition on small degrees."""
    rng = np.random.default_rng(0)
    for _ in range(5):
        ip, ix = random_graph(40, 0.2, rng)
        Pd = dense_P(ip, ix)
        p = oracle_partition(ip, ix, np.zeros(40, np.int32), 1, 0)
        np.testing.assert_array_equal(_dense_from_part(p, 40), Pd)


def test_split_worked_examples():
    ex = G["split_two_nodes"]
    ip, ix = csr_from_edges(2, ex["edges"])
    for m in range(2):
        p = oracle_partition(ip, ix, np.array(ex["part_of"], np.int32), 2, m)
        assert list(p.halo_ids) == ex["halo"][m]
        assert p.col.tolist() == [0, 1] and p.val.tolist() == [0.5, 0.5]  # P_in=[[.5]], P_out=[[.5]]
    ex = G["split_path"]
    ip, ix = csr_from_edges(3, ex["edges"])
    p = oracle_partition(ip, ix, np.array(ex["part_of"], np.int32), 2, 0)
    assert list(p.halo_ids) == ex["halo0"]
    row1 = slice(p.row_ptr[1], p.row_ptr[2])
    halo_entries = [v for c, v in zip(p.col[row1], p.val[row1]) if c >= p.n_local]
    assert len(halo_entries) == 1 and abs(halo_entries[0] - ex["P_out_row1"]) < 1e-7


def test_m1_has_empty_halo():
    rng = np.random.default_rng(1)
    ip, ix = random_graph(30, 0.2, rng)
    p = oracle_partition(ip, ix, np.zeros(30, np.int32), 1, 0)
    assert p.n_halo == 0 and p.send_idx.size == 0 and p.nnz == ix.size + 30


def test_k4_halo_ratio():
    ex = G["halo_ratio_k4"]
    ip, ix = csr_from_edges(ex["n"], ex["edges"])
    for m in range(2):
        p = oracle_partition(ip, ix, np.array(ex["part_of"], np.int32), 2, m)
        assert p.n_halo / p.n_local == ex["ratio"]


@pytest.mark.parametrize("seed", range(50))
def test_reconstruction_and_brute_force(seed):
    """S:116/S:152 zero-tolerance reconstruction; bit-exact vs the brute-force loops."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(5, 48))
    ip, ix = random_graph(n, float(rng.uniform(0.05, 0.4)), rng)
    M = int(rng.integers(1, 5))
    part = random_parts(n, M, rng)
    Pd = dense_P(ip, ix)
    covered = np.zeros(n, int)
    for m in range(M):
        p = oracle_partition(ip, ix, part, M, m)
        covered[p.local_ids] += 1
        np.testing.assert_array_equal(_dense_from_part(p, n), Pd[p.local_ids])
        assert np.all(p.col[p.row_ptr[:-1][np.diff(p.row_ptr) > 0]] >= 0)
        b = brute_partition(ip, ix, part, M, m)
        assert p.local_ids.tolist() == b["V"] and p.halo_ids.tolist() == b["H"]
        assert p.row_ptr.tolist() == b["row_ptr"] and p.col.tolist() == b["col"]
        assert p.val.tolist() == [np.float32(v) for v in b["val"]]
        assert p.send_idx.tolist() == b["send"] and p.send_count.tolist() == b["send_count"]
        assert p.recv_count.tolist() == b["recv_count"]
        assert p.rh_ptr.tolist() == b["rh_ptr"] and p.rh_col.tolist() == b["rh_col"]
        assert p.rh_val.tolist() == [np.float32(v) for v in b["rh_val"]]
        # in-block entries precede halo entries in every row
        for i in range(p.n_local):
            c = p.col[p.row_ptr[i]:p.row_ptr[i + 1]]
            assert np.all(np.diff(c) > 0)
    assert np.all(covered == 1)  # S:153 disjoint cover


@pytest.mark.parametrize("seed", range(10))
def test_send_lists_match_peer_halo_segments(seed):
    """S_{m->k} (sender m) equals the owner-m segment of H_k (receiver k), in order."""
    rng = np.random.default_rng(200 + seed)
    n = int(rng.integers(10, 60))
    ip, ix = random_graph(n, 0.15, rng)
    M = int(rng.integers(2, 6))
    part = random_parts(n, M, rng)
    parts = [oracle_partition(ip, ix, part, M, m) for m in range(M)]
    tot_s = tot_r = 0
    for m, pm in enumerate(parts):
        for k, pk in enumerate(parts):
            if k == m:
                assert pm.send_count[m] == 0
                continue
            s = pm.send_idx[pm.send_off[k]:pm.send_off[k] + pm.send_count[k]]
            seg = pk.halo_ids[pk.recv_off[m]:pk.recv_off[m] + pk.recv_count[m]]
            np.testing.assert_array_equal(pm.local_ids[s], seg)
        tot_s += pm.send_count.sum()
        tot_r += pm.recv_count.sum()
    assert tot_s == tot_r


def test_halo_ratio_independent_recount():
    rng = np.random.default_rng(5)
    ip, ix = random_graph(60, 0.1, rng)
    part = random_parts(60, 3, rng)
    deg = degrees(ip)
    for m in range(3):
        p = oracle_partition(ip, ix, part, 3, m)
        hs = set()
        for v in range(60):
            if part[v] == m:
                for u in ix[ip[v]:ip[v] + deg[v]]:
                    if part[u] != m:
                        hs.add(int(u))
        assert p.n_halo == len(hs)


def test_invalid_partitions_raise():
    ip, ix = csr_from_edges(3, [(0, 1)])
    with pytest.raises(ValueError):
        oracle_partition(ip, ix, np.array([0, 0, 0], np.int32), 2, 0)  # empty part
    with pytest.raises(ValueError):
        oracle_partition(ip, ix, np.array([0, 1, 2], np.int32), 4, 0)
