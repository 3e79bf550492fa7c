"""CPU oracle for the SFSeg / SFSeg++ power-iteration hot path (TEST INFRASTRUCTURE).

This package is test infrastructure only.  It may be imported, called or
executed ONLY by ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs.  The product path
(``paper_2212_08058_b200``) never imports it and shares no code with it.

It is a plain, slow, float64 numpy transcription of the paper's definitions
(arxiv 2212.08058, /root/reference/PAPER.md) -- see ``sfseg_oracle.py`` for the
per-function citations and ``dense.py`` for the explicit adjacency matrix used
to pin it.  Pins live in ``tests/test_oracle_pins.py``.

Parity status per function:
  gaussian_taps          pinned (SPEC worked value S:118, closed-form sums)
  combine                pinned (SPEC worked values S:187-189)
  gaussian_filter        pinned (direct triple loop, impulse response, dense M)
  power_iterate          pinned (dense M brute force, eigh closed form, PF invariants)
  normalize_l2           pinned
  threshold              parity unpinned beyond its definition (SURVEY A12 reading)
  power_iterate_backward pinned (central finite differences, Euler identity)
  full.full_step / power_iterate_full (Eq.7 with p, alpha and
                         a pairwise map) pinned (entry-by-entry Eq.2 matrix, SPEC
                         closed forms S:196-198, reduction to the hot path)
"""
from .sfseg_oracle import (  # noqa: F401
    ACT_IDENTITY, ACT_SIGMOID, THR_PER_FRAME_MAX, THR_GLOBAL_MAX, THR_ABSOLUTE,
    DegenerateError, gaussian_taps, combine, correlate_axis, gaussian_filter,
    apply_M, normalize_l2, power_iterate, threshold, power_iterate_backward, soft_binarize,
    binarize_kappa,
)
from .full import full_step, combine_full, power_iterate_full  # noqa: F401,E402
from .dense import dense_M_taylor  # noqa: F401,E402
from .online import window_starts, power_iterate_online  # noqa: F401,E402
from .learn import AdamW, mse_loss_grad, focal_dice_loss_grad, train  # noqa: F401,E402
