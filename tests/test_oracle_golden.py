"""Pin the CPU oracle against vectors produced by the reference itself.

tests/golden/*.npz were written by tests/golden/make_golden.py, which runs
the reference package (fluidrank) on these inputs.  The oracle must match
bit for bit: same CSR, same history/rank vectors, same counters.
"""

import numpy as np
import pytest

KINDS = ("sweep", "max", "per", "op", "op2")


def test_csr_cases_bit_exact(golden_csr, oracle):
    for k in range(int(golden_csr["count"])):
        n = int(golden_csr[f"c{k}_n"])
        off, tgt, stats = oracle.csr_build(n, golden_csr[f"c{k}_src"], golden_csr[f"c{k}_dst"],
                                           clean=bool(golden_csr[f"c{k}_clean"]))
        assert np.array_equal(off, golden_csr[f"c{k}_off"]), k
        assert np.array_equal(tgt, golden_csr[f"c{k}_tgt"]), k
        assert tuple(stats) == tuple(golden_csr[f"c{k}_stats"]), k


def test_csr_strict_errors_match_reference(golden_csr, oracle):
    for j in range(int(golden_csr["bad_count"])):
        with pytest.raises(ValueError) as err:
            oracle.csr_build(int(golden_csr[f"bad{j}_n"]), golden_csr[f"bad{j}_src"], golden_csr[f"bad{j}_dst"])
        assert str(err.value) == str(golden_csr[f"bad{j}_msg"])


@pytest.mark.parametrize("kind", KINDS)
def test_sequential_runs_bit_exact(golden_small, oracle, kind):
    for tag in golden_small["tags"]:
        tag = str(tag)
        off, tgt = golden_small[f"{tag}_off"], golden_small[f"{tag}_tgt"]
        tel = golden_small[f"{tag}_teleport"] if f"{tag}_teleport" in golden_small else None
        r = oracle.run_seq(off, tgt, float(golden_small[f"{tag}_damping"]),
                           float(golden_small[f"{tag}_target_error"]), kind, teleport=tel)
        assert np.array_equal(r.rank, golden_small[f"{tag}_{kind}_rank"]), tag
        assert np.array_equal(r.history, golden_small[f"{tag}_{kind}_history"]), tag
        diffusions, steps, rows = golden_small[f"{tag}_{kind}_counts"]
        assert (r.diffusions, r.elementary_steps, len(r.trace)) == (diffusions, steps, rows), tag
        assert r.residual == float(golden_small[f"{tag}_{kind}_residual"]), tag


def test_power_iteration_bit_exact(golden_small, oracle):
    for tag in golden_small["tags"]:
        tag = str(tag)
        off, tgt = golden_small[f"{tag}_off"], golden_small[f"{tag}_tgt"]
        tel = golden_small[f"{tag}_teleport"] if f"{tag}_teleport" in golden_small else None
        x, iters, _ = oracle.power_iterate(off, tgt, float(golden_small[f"{tag}_damping"]),
                                           float(golden_small[f"{tag}_target_error"]), teleport=tel)
        assert np.array_equal(x, golden_small[f"{tag}_mat_iter_rank"]), tag
        assert iters == int(golden_small[f"{tag}_mat_iter_iters"]), tag


@pytest.mark.parametrize("tag", ["cfg1", "web5k"])
def test_config_graphs(golden_configs, oracle, tag):
    """BASELINE config 1 and a scaled config 2: generator, clean CSR, sweep rank."""
    n, seed = int(golden_configs[f"{tag}_n"]), int(golden_configs[f"{tag}_seed"])
    cfg = oracle.uniform_config(10) if tag == "cfg1" else oracle.web_config(8.0)
    src, dst = oracle.gen_edges(cfg, n, seed)
    assert np.array_equal(src, golden_configs[f"{tag}_src"])
    assert np.array_equal(dst, golden_configs[f"{tag}_dst"])
    off, tgt, stats = oracle.csr_build(n, src, dst, clean=True)
    assert np.array_equal(off, golden_configs[f"{tag}_off"])
    assert np.array_equal(tgt, golden_configs[f"{tag}_tgt"])
    assert tuple(stats) == tuple(golden_configs[f"{tag}_stats"])
    r = oracle.run_seq(off, tgt, 0.85, float(golden_configs[f"{tag}_target_error"]), "sweep")
    assert np.array_equal(r.rank, golden_configs[f"{tag}_sweep_rank"])
    assert r.diffusions == int(golden_configs[f"{tag}_sweep_counts"][0])
