"""Device generator and CSR construction: bit-exact against the oracle and the reference goldens."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def to_np(t):
    return t.cpu().numpy()


def test_csr_golden_cases(cuda, golden_csr):
    for k in range(int(golden_csr["count"])):
        n = int(golden_csr[f"c{k}_n"])
        off, tgt, stats = cuda.csr_build(n, golden_csr[f"c{k}_src"], golden_csr[f"c{k}_dst"],
                                         clean=bool(golden_csr[f"c{k}_clean"]))
        assert np.array_equal(to_np(off), golden_csr[f"c{k}_off"]), k
        assert np.array_equal(to_np(tgt).astype(np.uint32), golden_csr[f"c{k}_tgt"]), k
        assert tuple(stats) == tuple(golden_csr[f"c{k}_stats"]), k


def test_csr_errors_match_reference_messages(cuda, golden_csr):
    for j in range(int(golden_csr["bad_count"])):
        with pytest.raises(ValueError) as err:
            cuda.SparseGraph.from_edges(int(golden_csr[f"bad{j}_n"]), golden_csr[f"bad{j}_src"],
                                        golden_csr[f"bad{j}_dst"])
        assert str(err.value) == str(golden_csr[f"bad{j}_msg"])
    with pytest.raises(ValueError, match="out of range"):
        cuda.SparseGraph.from_edges(3, [0, -1], [1, 2])


def test_empty_and_edgeless(cuda):
    g = cuda.SparseGraph.from_edges(3, [], [])
    assert g.edge_count == 0 and g.dangling_count == 3
    assert to_np(g.out_offsets).tolist() == [0, 0, 0, 0]


@pytest.mark.parametrize("n,seed", [(5000, 1), (70000, 2)])
def test_web_generator_bit_exact(cuda, oracle, n, seed):
    from paper_1202_6158_b200 import gen
    src, dst = gen.generate_edges(gen.web_config(8.0), n, seed)
    osrc, odst = oracle.gen_edges(oracle.web_config(8.0), n, seed)
    assert np.array_equal(to_np(src).astype(np.uint32), osrc)
    assert np.array_equal(to_np(dst).astype(np.uint32), odst)
    off, tgt, stats = cuda.csr_build(n, src, dst, clean=True)
    ooff, otgt, ostats = oracle.csr_build(n, osrc, odst, clean=True)
    assert np.array_equal(to_np(off), ooff)
    assert np.array_equal(to_np(tgt).astype(np.uint32), otgt)
    assert tuple(stats) == tuple(ostats)


def test_uniform_generator_bit_exact(cuda, oracle, golden_configs):
    from paper_1202_6158_b200 import gen
    src, dst = gen.generate_edges(gen.uniform_config(10), 10_000, 1234)
    assert np.array_equal(to_np(src).astype(np.uint32), golden_configs["cfg1_src"])
    assert np.array_equal(to_np(dst).astype(np.uint32), golden_configs["cfg1_dst"])
    g, rep = gen.generate(gen.uniform_config(10), 10_000, 1234)
    assert np.array_equal(to_np(g.out_offsets), golden_configs["cfg1_off"])
    assert np.array_equal(to_np(g.out_targets).astype(np.uint32), golden_configs["cfg1_tgt"])


def test_shuffled_edges_and_every_sort_bin(cuda, oracle):
    """Rows of degree 1..16 (thread), 17..1024 (warp), 1025..49152 (block), >49152 (global)."""
    rng = np.random.default_rng(0)
    n = 120_000
    degs = {0: 60_000, 1: 5, 2: 20, 3: 3000, 4: 50_000, 5: 200_000, 6: 17, 7: 1024, 8: 1025, 9: 49_152, 10: 49_153}
    src, dst = [], []
    for s, d in degs.items():
        t = rng.choice(n - 1, size=min(d, n - 1), replace=False)
        t = t + (t >= s)
        src.append(np.full(t.size, s))
        dst.append(t)
    extra = rng.integers(0, n, size=(300_000, 2))
    extra = extra[extra[:, 0] != extra[:, 1]]
    src.append(extra[:, 0])
    dst.append(extra[:, 1])
    src = np.concatenate(src)
    dst = np.concatenate(dst)
    # duplicate some edges inside the big rows and add self-loops for the clean path
    dup = rng.integers(0, src.size, 20_000)
    csrc = np.concatenate([src, src[dup], np.arange(50)])
    cdst = np.concatenate([dst, dst[dup], np.arange(50)])
    perm = rng.permutation(csrc.size)
    csrc, cdst = csrc[perm], cdst[perm]
    off, tgt, stats = cuda.csr_build(n, csrc, cdst, clean=True)
    ooff, otgt, ostats = oracle.csr_build(n, csrc, cdst, clean=True)
    assert np.array_equal(to_np(off), ooff)
    assert np.array_equal(to_np(tgt).astype(np.uint32), otgt)
    assert tuple(stats) == tuple(ostats)
    # strict path on the clean set rejects nothing and gives the same CSR
    s2 = np.repeat(np.arange(n), np.diff(ooff))
    perm = rng.permutation(s2.size)
    g = cuda.SparseGraph.from_edges(n, s2[perm], otgt.astype(np.int64)[perm])
    assert np.array_equal(to_np(g.out_offsets), ooff)
    assert np.array_equal(to_np(g.out_targets).astype(np.uint32), otgt)
    with pytest.raises(ValueError, match="duplicate edge in edge arrays"):
        cuda.SparseGraph.from_edges(n, np.append(s2, 5), np.append(otgt, otgt[ooff[5]]))


def test_in_degree_and_reverse_csr(cuda, oracle):
    osrc, odst = oracle.gen_edges(oracle.web_config(8.0), 30_000, 4)
    g = cuda.SparseGraph.from_edges_clean(30_000, osrc, odst)
    off, tgt = g.host_csr()
    assert np.array_equal(to_np(g.in_degree), np.bincount(tgt, minlength=g.n))
    in_off, in_src = g.reverse_csr()
    o_in_off, o_in_src = oracle.transpose(g.n, off, tgt.astype(np.uint32))
    assert np.array_equal(to_np(in_off), o_in_off)
    assert np.array_equal(to_np(in_src).astype(np.uint32), o_in_src)


def test_load_edge_list_matches_reference_semantics(cuda):
    import io
    g = cuda.load_edge_list(io.StringIO("0 1\n0 1\n1 1\n"))
    assert g.n == 2 and g.edge_count == 1 and g.dangling_count == 1
    assert g.report.duplicates_dropped == 1 and g.report.self_loops_dropped == 1
    g = cuda.load_edge_list(io.StringIO("n 10 http://a\nn 20 http://b\nn 30\ne 10 20\ne 20 30\n"))
    assert g.n == 3 and g.edge_count == 2 and g.labels[0] == "http://a" and g.original_ids == [10, 20, 30]
    g = cuda.load_edge_list(io.StringIO("5 3\n3 7\n"))
    assert g.original_ids == [5, 3, 7] and g.has_edge(0, 1) and g.has_edge(1, 2)


def test_apply_delta_and_delta_columns(cuda):
    g = cuda.SparseGraph.from_edges(2, [0, 1], [1, 0])
    g2 = cuda.apply_delta(g, cuda.GraphDelta(added=[], removed=[(1, 0)]))
    assert g2.dangling.tolist() == [1]
    g3 = cuda.apply_delta(g2, cuda.GraphDelta(added=[(1, 0)], removed=[]))
    assert to_np(g3.out_targets).tolist() == to_np(g.out_targets).tolist()
    assert cuda.delta_columns(g, g2) == [1]
    assert cuda.delta_columns(g, g3) == []
    with pytest.raises(cuda.DeltaError):
        cuda.apply_delta(g, cuda.GraphDelta(added=[(0, 1)], removed=[]))


@pytest.mark.parametrize("kind,n,seed", [("uniform", 10_000, 1234), ("web8", 70_000, 2), ("web16", 300_000, 0)])
def test_exact_size_generator_bit_exact(cuda, oracle, kind, n, seed):
    """gen.generate(exact=True) -- base draw, cleaned, then fill rounds redrawing the dropped
    slots on the device -- is bit-exact with the oracle's gen_graph_exact, report included."""
    from paper_1202_6158_b200 import gen
    g, rep = gen.generate({"uniform": gen.uniform_config(10), "web8": gen.web_config(8.0),
                           "web16": gen.web_config(16.0)}[kind], n, seed, exact=True)
    ocfg = {"uniform": oracle.uniform_config(10), "web8": oracle.web_config(8.0),
            "web16": oracle.web_config(16.0)}[kind]
    off, tgt, orep = oracle.gen_graph_exact(ocfg, n, seed)
    assert np.array_equal(to_np(g.out_offsets), off)
    assert np.array_equal(to_np(g.out_targets).astype(np.uint32), tgt)
    assert (rep.slots, rep.realized_links, rep.duplicates, rep.self_loops, rep.target_links, rep.rounds,
            rep.unfilled) == (orep["slots"], orep["realized_links"], orep["duplicates"], orep["self_loops"],
                              orep["target_links"], orep["rounds"], orep["unfilled"])
