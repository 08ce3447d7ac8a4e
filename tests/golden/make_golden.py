"""Generate tests/golden/*.npz from the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

The fixtures pin the CPU oracle (oracle/fr_oracle.c) and, through it, the
CUDA product.  Everything is produced by the reference package's own public
API (fluidrank.graph / engine / sched / baseline / gen); the only input not
produced by the reference is the BASELINE config-1/config-2 edge lists, which
come from the generator specification in the oracle and are then cleaned and
ranked by the reference.  Nothing here is read at test time except the .npz
outputs.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from fluidrank import baseline, engine, gen, graph, sched  # noqa: E402

from oracle import oracle as O  # noqa: E402

KINDS = ("sweep", "max", "per", "op", "op2")


def random_graph(rng, n, max_out=4, dangling_frac=0.3):
    """Same construction as the reference tests' conftest.random_graph."""
    dangling = rng.random(n) < dangling_frac
    src, dst = [], []
    for j in range(n):
        if dangling[j]:
            continue
        k = min(int(rng.integers(1, max_out + 1)), n - 1)
        targets = rng.choice(n - 1, size=k, replace=False)
        targets = targets + (targets >= j)
        src.extend([j] * k)
        dst.extend(int(t) for t in targets)
    if not src:
        src, dst = [0], [1]
    return graph.SparseGraph.from_edges(n, src, dst)


def csr_cases():
    """from_edges / build_clean_edges on shuffled edge lists (graph.py:74-200)."""
    rng = np.random.default_rng(2024)
    out = {}
    k = 0
    for trial in range(12):
        n = int(rng.integers(2, 400))
        m = int(rng.integers(1, 6 * n))
        src = rng.integers(0, n, m)
        dst = rng.integers(0, n, m)
        s2, d2, dups, loops = graph.build_clean_edges(src, dst)
        g = graph.SparseGraph.from_edges(n, s2, d2)
        out[f"c{k}_n"] = np.int64(n)
        out[f"c{k}_src"] = src.astype(np.uint32)
        out[f"c{k}_dst"] = dst.astype(np.uint32)
        out[f"c{k}_off"] = g.out_offsets
        out[f"c{k}_tgt"] = g.out_targets.astype(np.uint32)
        out[f"c{k}_stats"] = np.array([g.edge_count, dups, loops], dtype=np.int64)
        out[f"c{k}_clean"] = np.int64(1)
        k += 1
        # the clean edge set, shuffled, must also pass the strict path
        perm = rng.permutation(s2.size)
        out[f"c{k}_n"] = np.int64(n)
        out[f"c{k}_src"] = s2[perm].astype(np.uint32)
        out[f"c{k}_dst"] = d2[perm].astype(np.uint32)
        out[f"c{k}_off"] = g.out_offsets
        out[f"c{k}_tgt"] = g.out_targets.astype(np.uint32)
        out[f"c{k}_stats"] = np.array([g.edge_count, 0, 0], dtype=np.int64)
        out[f"c{k}_clean"] = np.int64(0)
        k += 1
    # strict-mode rejections, with the reference's messages
    bad = [(3, [0, 1], [1, 3]), (3, [0, 1], [1, 1]), (3, [0, 0, 1], [1, 1, 2])]
    for j, (n, s, d) in enumerate(bad):
        try:
            graph.SparseGraph.from_edges(n, s, d)
            msg = ""
        except ValueError as exc:
            msg = str(exc)
        out[f"bad{j}_n"] = np.int64(n)
        out[f"bad{j}_src"] = np.array(s, dtype=np.uint32)
        out[f"bad{j}_dst"] = np.array(d, dtype=np.uint32)
        out[f"bad{j}_msg"] = np.array(msg)
    out["count"] = np.int64(k)
    out["bad_count"] = np.int64(len(bad))
    return out


def run_case(out, tag, g, target_error, teleport=None, kinds=KINDS, damping=0.85):
    out[f"{tag}_off"] = g.out_offsets
    out[f"{tag}_tgt"] = g.out_targets.astype(np.uint32)
    out[f"{tag}_target_error"] = np.float64(target_error)
    out[f"{tag}_damping"] = np.float64(damping)
    if teleport is not None:
        out[f"{tag}_teleport"] = np.asarray(teleport, dtype=np.float64)
    params = engine.DiffusionParams(damping=damping, teleport=teleport, target_error=target_error)
    for kind in kinds:
        state = engine.init(g, params)
        rank, trace = engine.run(g, params, sched.make_scheduler(kind), state=state)
        out[f"{tag}_{kind}_rank"] = rank
        out[f"{tag}_{kind}_history"] = state.history
        out[f"{tag}_{kind}_counts"] = np.array([state.diffusions, state.elementary_steps, len(trace.rows)],
                                               dtype=np.int64)
        out[f"{tag}_{kind}_residual"] = np.float64(state.residual)
    x, trace = baseline.power_iterate(g, params)
    out[f"{tag}_mat_iter_rank"] = x
    out[f"{tag}_mat_iter_iters"] = np.int64(trace.rows[-1].diffusions)


def small_runs():
    """engine.run for every deterministic scheduler + power_iterate (engine.py:240, baseline.py:20)."""
    out = {}
    tags = []
    G = graph.SparseGraph.from_edges
    fixtures = {
        "two_cycle": (G(2, [0, 1], [1, 0]), None),
        "chain": (G(2, [0], [1]), None),
        "star": (G(5, [0, 0, 0, 0], [1, 2, 3, 4]), None),
        "isolated3": (G(3, [], []), np.array([0.2, 0.3, 0.5])),
    }
    for tag, (g, tel) in fixtures.items():
        run_case(out, tag, g, 1e-10, teleport=tel)
        tags.append(tag)
    rng = np.random.default_rng(77)
    for k in range(8):
        n = int(rng.integers(5, 200))
        g = random_graph(rng, n, dangling_frac=float(rng.uniform(0.0, 0.6)))
        tel = None
        if k % 3 == 2:
            tel = rng.random(n)
            tel /= tel.sum()
            tel[-1] = 1.0 - tel[:-1].sum()
            if abs(tel.sum() - 1.0) > 1e-12 or tel[-1] < 0:
                tel = None
        run_case(out, f"rg{k}", g, 1e-10 if k % 2 else 1e-9, teleport=tel)
        tags.append(f"rg{k}")
    # the paper's section-4.1 scenario generator (gen.py:66), two scaled scenarios
    for k, (n, links, alpha) in enumerate([(600, 1500, 2.0), (800, 5000, 1.5)]):
        g, _ = gen.generate(gen.GenConfig(n=n, links=links, alpha=alpha, seed=31 + k))
        run_case(out, f"paper{k}", g, 1e-9)
        tags.append(f"paper{k}")
    out["tags"] = np.array(tags)
    return out


def config_graphs():
    """BASELINE config 1 (10k uniform) and a scaled config-2 web graph.

    Edge lists come from the oracle's generator spec; cleaning, CSR and the
    ranks come from the reference (build_clean_edges + from_edges + run).
    """
    out = {}
    cases = {
        "cfg1": (O.uniform_config(10), 10_000, 1234, 1e-10),
        "web5k": (O.web_config(mean_degree=8.0), 5_000, 99, 1e-9),
    }
    for tag, (cfg, n, seed, te) in cases.items():
        src, dst = O.gen_edges(cfg, n, seed)
        s2, d2, dups, loops = graph.build_clean_edges(src.astype(np.int64), dst.astype(np.int64))
        g = graph.SparseGraph.from_edges(n, s2, d2)
        out[f"{tag}_n"] = np.int64(n)
        out[f"{tag}_seed"] = np.int64(seed)
        out[f"{tag}_src"] = src
        out[f"{tag}_dst"] = dst
        out[f"{tag}_stats"] = np.array([g.edge_count, dups, loops], dtype=np.int64)
        run_case(out, tag, g, te, kinds=("sweep",))
    return out


def main():
    np.savez_compressed(os.path.join(HERE, "csr_cases.npz"), **csr_cases())
    print("csr_cases done")
    np.savez_compressed(os.path.join(HERE, "small_runs.npz"), **small_runs())
    print("small_runs done")
    np.savez_compressed(os.path.join(HERE, "config_graphs.npz"), **config_graphs())
    print("config_graphs done")


if __name__ == "__main__":
    main()
