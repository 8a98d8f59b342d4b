"""ORACLE — test infrastructure only, never the product path.

A CPU float64 restatement of the reference's pack hot path
(`/root/reference/pkg/src/packtrain/{engine,data,packing}.py`), used as the
checker by `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs.  Nothing under
`paper_2002_02885_b200/` may import it; the product path fails loudly when
the CUDA library is missing instead of falling back here.

Pinning: every function cites the reference file:line it restates.  The
restatement is checked against (i) the reference's own known-answer tests
(`pkg/tests/test_engine.py`) re-evaluated in `tests/test_oracle.py`, and (ii)
golden vectors produced by importing the reference itself in the build
container (`tests/golden/make_golden.py` → `tests/golden/*.npz`).
"""
from .mlp64 import (ACTIVATIONS, OPTIMIZERS, OracleMember, epoch_order,
                    forward_backward, member_forward_loss, optimizer_step,
                    oracle_packed_step, oracle_standalone_step, seeded_rng,
                    synth_blobs, xavier_layers)

__all__ = [
    "ACTIVATIONS", "OPTIMIZERS", "OracleMember", "epoch_order",
    "forward_backward", "member_forward_loss", "optimizer_step",
    "oracle_packed_step", "oracle_standalone_step", "seeded_rng",
    "synth_blobs", "xavier_layers",
]
