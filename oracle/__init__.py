"""CPU oracle for the cuGenOpt evolve hot path — TEST INFRASTRUCTURE ONLY.

This package is a plain-Python/numpy restatement of the reference's algorithm
(`/root/reference/pkg/src/genopt/*`, cited per function as `file:line`).  It is
the checker the CUDA path is compared against, never the thing measured or
shipped: only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` leg may import it.  The product package
`paper_2603_19163_b200` must not import anything from here.

Pinning:
  * `tests/golden/make_golden.py` runs the unmodified reference (importable in
    the build container only) and freezes objective values, operator traces,
    AOS updates, population sizing and whole-run trajectories into
    `tests/golden/*.json`; `tests/test_oracle_golden.py` checks this oracle
    against every one of them, so the oracle is pinned to the reference.
  * The oracle engine takes a pluggable word source.  With the reference's own
    MT19937 streams (`rng.mt_stream`) it reproduces reference `run()` results
    bit-for-bit; with Philox4x32-10 streams (`rng.philox_stream`) it
    reproduces the GPU engine bit-for-bit on integer instances.  The draw
    ORDER is identical in both modes; only the 32-bit word generator differs.

Modules:
  rng       mix64, Philox4x32-10, CPython-exact random()/randrange()/shuffle()/sample()
  problems  objective / penalty restatements for the on-path problems
  moves     operator restatements (operators.py, demo_ops.py)
  aos       adaptive operator selection restatement (aos.py, profiles.py)
  engine    population init, sizing, islands, evolve_generation, run loop
"""
