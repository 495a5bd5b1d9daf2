"""Float64 CPU oracle for the deep-BSDE training hot path of arXiv:1910.11623.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_1910_11623_b200``) never imports it and
this package never imports the product: the two share no code.

Every function cites the passage of ``PAPER.md`` (P:<line>) it follows, or the
reading adopted in ``DESIGN.md`` §Readings (R<k>) where the paper is silent.

Modules
-------
philox        Philox4x32-10 counter-based generator and the Box-Muller map (R8).
bsde          per-step Z-net rollout, terminal loss, hand adjoint, Adam,
              multilevel prolongation, initialisation (Eq. 7, §3.2).
closed_forms  closed-form values the oracle is pinned against (heat optimum,
              Cole-Hopf for HJB, Allen-Cahn linearisation / zero-Z ODE limit).

Parity status: every function here is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py``; none is "parity unpinned".
"""
