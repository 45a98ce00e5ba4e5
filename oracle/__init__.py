"""ParaDySe oracle — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU (numpy fp64) implementation of what the
B200 hot path computes.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs may import it.  The
product path (``paper_2511_13198_b200``) never imports, links or executes
anything here, and this package never imports the product path.  The two share
no code; only the seeded input generators in ``synth/`` serve both.

Modules (each function cites the PAPER.md / SPEC.md passage it follows):
  layer       unsharded layer forward + backward (Eqs. 1-4 + north_star additions)
  grid        simulated 1D device grid: collectives, comm log, memory ledger
  shard       Table 2 "Specification" row layouts (spec-layout shards)
  strategies  MegatronTS / UlyssesZ / METP sharded simulations (fwd + bwd)
  memory      per-layer memory model (Eq. 6 reading, R-22)
  flops       FLOP / comm-byte model
  selector    Algorithm 1 step by step, pop_useless, brute force
  costmodel   Eq. 9 hybrid dispatch: exported random-forest evaluation, AIC poly
  layouts     Table 2 rows as data

Parity pins are listed per module header; "parity unpinned" marks the parts
without an independent pin.
"""
