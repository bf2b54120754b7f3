"""CPU oracle for the CRL critic hot path (arXiv 2408.11052, "JaxGCRL").

TEST INFRASTRUCTURE ONLY.  This package is the plain, slow, obviously-correct fp64
(NumPy) restatement of what the hot path computes, written from PAPER.md.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import it.  The product path (``paper_2408_11052_b200``)
never imports it, and it never imports the product path: the two share no code.

Citations: ``P:NNN`` is a line of /root/reference/PAPER.md (section named alongside);
``A-NN`` / ``C-N`` are the readings and contract items listed in DESIGN.md §3.

Modules
  philox   Philox4x32-10 counter-based generator (A-18; pinned by Random123 KAT vectors)
  replay   trajectory buffer + hindsight relabeling (Alg.1)
  mlp      phi / psi encoders forward + backward (Table 2)
  energy   critic energies L2 / dot / cos and their VJPs (App. A.2)
  losses   InfoNCE fwd / bwd / sym + logsumexp penalty and dL/dlogits
  adam     bias-corrected Adam (A-15; Alg.1, Table 2)
  critic   the whole critic step (Alg.1) and the actor loss (Eq.3)

Parity status: every function here is pinned by a ``-m "not gpu"`` test in
tests/test_oracle_*.py against closed forms, invariants, finite differences or brute
force (see DESIGN.md §3 "Pins").  No function is "parity unpinned".
"""
