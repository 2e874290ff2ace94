"""CPU oracle for the Ripples P-Reduce hot path (arXiv 1909.08029).

TEST INFRASTRUCTURE ONLY. Nothing in the product path (``paper_1909_08029_b200``)
may import, call or execute this package; only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs do. It shares no code with the CUDA/C++ library:
the only common module is ``rp_inputs`` (the seeded input generator, which
holds none of the method's arithmetic).

Plain, slow, sequential NumPy. Each function cites the PAPER.md passage
(``P:<line>``, section / algorithm label) it follows. Where the paper is silent
the reading of SURVEY.md §8(c) c.2 is taken; every reading is listed in
DESIGN.md "Readings of the paper".

Modules and what pins them (tests/test_oracle_*.py, all ``-m "not gpu"``):

  algebra   W (pairwise), F^G, X·W in fp64
            pins: paper's n=5 worked examples, doubly stochastic,
            (F^G)^T F^G = F^G, fused-pair product
  update    SGD step + P-Reduce, pinned fp32 order    alg1
            pins: X·F^G closed form (fp64 library matmul), k=2 exact-halving
            identity, singleton = SGD within 1 ulp, mass conservation,
            idempotence, G = all = global mean, exact rational replay
            bf16 replicas (reading R26): bf16_round pinned to hand-derived
            IEEE ties (tests/golden/bf16_rne_ties.txt) and torch's RNE
            conversion; update = fp32 update rounded once; half-ulp bound
  schedule  static rules PAPER4 and SHIFT_K
            pins: P:879 printed facts, fig:scheduler table, exhaustive
            disjointness / coverage / union-find connectivity
  gg        Group Buffer + Global Division + filter
            pins: fig:global_devision walk-through, filter
            rule, brute-force interleavings (conflict-freedom,
            GB depth, no deadlock), uniform membership frequency
  sim       lockstep simulator and async trace replay alg1
            pins: exact-arithmetic (fractions) replay of small runs

Parity unpinned: none of the functions above. (Throughput has no paper number:
see DESIGN.md §Measurement.)
"""
from . import algebra, update, schedule, gg, sim  # noqa: F401
