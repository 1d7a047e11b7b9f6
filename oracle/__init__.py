"""CPU ORACLE for the local-smoothing adaptive GMG hot path (arXiv 1904.03317).

*** TEST INFRASTRUCTURE ONLY. ***  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import
anything under ``oracle/``.  The product path (``paper_1904_03317_b200``) never
imports it and fails loudly when its CUDA library is missing.

Plain, slow, obviously correct numpy/scipy code, fp64 throughout, every
function citing the PAPER.md passage (P:line) it follows.  It assembles the
level matrices explicitly (scipy.sparse CSR) and runs the paper's V-cycle
 with the local-smoothing block structure literally in
level-cell storage; ``oracle.abstract`` is an independent dense implementation
of the same algorithm on the level spaces V_l with hanging-node elimination,
used to pin this one.  Shares no code with the CUDA path.

Modules
  forest     forest of trees, Morton SFC, refinement recipes, 2:1 vertex closure
  partition  SFC leaf partition, first-child rule, efficiency model, ghost children
  spaces     level DoF sets D_l, classes S/E/B, numbering, lambda map, leaf DoFs
  fem        1-D Q_k matrices, element matrices, CSR level/leaf/transfer matrices
  mg         Chebyshev-Jacobi, eigenvalue estimate, coarse solve, V-cycle, CG
  abstract   dense V_l = V^S + V^I + V^L checker (P:413-458 literally)

"Parity unpinned" functions: none at the sizes the tests use; see DESIGN.md.
"""
