"""Node-selection rules, lifted from single nodes to whole-frontier sweeps.

Mirrors pkg/src/fluidrank/sched.py.  The reference picks one node per step;
on the GPU each sweep diffuses every node that satisfies the rule at once
(PAPER sec. 4.2: "in one iteration all i such that (F_n)_i is above a
threshold are all chosen, then scaling down the threshold progressively").
Every rule stays fair, so the limit is the same (PAPER Theorem 3.1-3.2):

  kind   reference rule (sched.py)               device sweep rule
  sweep  index-order passes, f >= theta          all nodes with |f| >= theta
  max    argmax f                                |f| >= decay * max|f|
  per    n mod N                                 every node holding fluid
  rand   uniform random node                     each node w.p. rand_frac
  op     argmax f/((in+1)(out+1))                |f| * w >= theta, same w
  op2    argmax f/(out+1)                        |f| * w >= theta, same w

The sweep rule also takes a degree exponent beta: score = |f| * (out+1)^-beta
(PAPER sec. 4.3: the cost of diffusing a node is proportional to #out).  On the
config-5 generator, beta = 0.5 with theta decaying 0.9 per sweep diffuses 32%
fewer edges than plain |f| (oracle run_psweep, N=1M), fewer than the
sequential reference itself.

next()/scores() keep the reference's single-node semantics for callers that
drive diffuse() themselves.
"""

from __future__ import annotations

import torch

from . import _lib

KINDS = ("max", "rand", "per", "sweep", "op", "op2")
POLICIES = ("exhaust", "geometric", "adaptive")
KERNEL_PATHS = ("fused", "binned", "owned")  # fr_solver_config.kernel_path 0, 1, 2


class DeviceSchedule:
    """A selection rule plus its theta policy; consumed by engine.run."""

    def __init__(self, kind, seed=0, decay=0.5, policy="exhaust", rand_frac=0.25,
                 edge_frac=0.2, thread_max_degree=0, block_min_degree=0, kernel_path="owned", hot_slots=0,
                 warm_slots=0, degree_exponent=0.0):
        if kind not in KINDS:
            raise ValueError(f"unknown scheduler kind {kind!r}; expected one of {KINDS}")
        if not 0.0 < decay < 1.0:
            raise ValueError(f"decay must be in (0, 1), got {decay}")
        if policy not in POLICIES:
            raise ValueError(f"unknown theta policy {policy!r}; expected one of {POLICIES}")
        self.kind = kind
        self.seed = int(seed)
        self.decay = float(decay)
        self.policy = policy
        self.rand_frac = float(rand_frac)
        if edge_frac <= 0:
            raise ValueError(f"edge_frac must be > 0, got {edge_frac}")
        self.edge_frac = float(edge_frac)
        self.thread_max_degree = int(thread_max_degree)
        self.block_min_degree = int(block_min_degree)
        if kernel_path not in KERNEL_PATHS:
            raise ValueError(f"kernel_path must be one of {KERNEL_PATHS}, got {kernel_path!r}")
        self.kernel_path = kernel_path
        self.hot_slots = int(hot_slots)
        self.warm_slots = int(warm_slots)
        if degree_exponent < 0:
            raise ValueError(f"degree_exponent must be >= 0, got {degree_exponent}")
        self.degree_exponent = float(degree_exponent)
        self._per_count = 0
        self._rng = None

    # -- device configuration ------------------------------------------
    def needs_weights(self):
        # op2's weight 1/(out+1) is computed on the device from the degree
        return self.kind == "op"

    def weights(self, graph):
        """Static score multipliers 1/((in+1)(out+1)) or 1/(out+1) (sched.py:131-138)."""
        w = (graph.out_degree + 1).to(torch.float64)
        if self.kind == "op":
            w = w * (graph.in_degree + 1).to(torch.float64)
        return 1.0 / w

    def solver_config(self, params, fluid_fp32=False, max_sweeps=0, max_diffusions=None):
        c = _lib.SolverConfig()
        c.damping = float(params.damping)
        c.target_error = float(params.target_error)
        c.decay = self.decay
        c.rand_frac = self.rand_frac
        c.edge_frac = self.edge_frac
        c.max_sweeps = int(max_sweeps or 0)
        c.max_diffusions = int(max_diffusions or 0)
        c.select = _lib.SELECT[self.kind]
        c.policy = _lib.POLICY[self.policy]
        c.fluid_fp32 = int(bool(fluid_fp32))
        c.thread_max_degree = self.thread_max_degree
        c.block_min_degree = self.block_min_degree
        c.seed = self.seed & 0xFFFFFFFF
        c.kernel_path = KERNEL_PATHS.index(self.kernel_path)
        c.hot_slots = self.hot_slots
        c.warm_slots = self.warm_slots
        c.degree_exponent = self.degree_exponent
        return c

    # -- reference single-node interface -------------------------------
    def scores(self, state, graph):
        """The per-node quantity the rule ranks (sched.py score_table)."""
        mag = state.fluid_magnitude().to(torch.float64)
        if self.kind in ("per", "rand"):
            return torch.full((graph.n,), 1.0 / graph.n, dtype=torch.float64, device=mag.device)
        if self.kind in ("op", "op2"):
            return mag * self.weights(graph)
        if self.degree_exponent:
            return mag * (graph.out_degree + 1).to(torch.float64) ** -self.degree_exponent
        return mag.clone()

    def next(self, state, graph):
        """One node, with the reference's tie-break (lowest index)."""
        if self.kind == "per":
            i = self._per_count % graph.n
            self._per_count += 1
            return i
        if self.kind == "rand":
            if self._rng is None:
                self._rng = torch.Generator().manual_seed(self.seed)
            return int(torch.randint(0, graph.n, (1,), generator=self._rng))
        s = self.scores(state, graph)
        return int(torch.argmax(s))  # first maximal index


def make_scheduler(kind, seed=0, sweep_decay=0.5, **kwargs):
    """Scheduler for a CLI kind token (sched.py:147-161)."""
    return DeviceSchedule(kind, seed=seed, decay=sweep_decay, **kwargs)


# reference class names
def GreedyScheduler():
    return DeviceSchedule("max")


def RandomScheduler(seed=0, chunk=4096):
    return DeviceSchedule("rand", seed=seed)


def RoundRobinScheduler():
    return DeviceSchedule("per")


def ThresholdSweepScheduler(decay=0.5):
    return DeviceSchedule("sweep", decay=decay)


def DegreeScaledScheduler(use_in_degree=True):
    return DeviceSchedule("op" if use_in_degree else "op2")
