"""Test-infrastructure ORACLE for the topology-based transient analysis of
arxiv 1409.7166 ("An Efficient Topology-Based Algorithm for Transient Analysis
of Power Grid", PAPER.md).

THIS PACKAGE IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import, call, link or execute anything here.  The
product path (``paper_1409_7166_b200``) never imports it, and this package never
imports the product.  The only module both sides use is the seeded input
generator ``gridgen`` (raw element values, none of the method's arithmetic).

Contents (each function cites the PAPER.md passage it follows):

* ``netlist``  - the circuit in the paper's §III notation: trivial nodes, source
  nodes, branches grouped by kind (Eq. (6)), built from generator output.
* ``pwl``      - piecewise-linear load currents (§II-A "modeled as piecewise
  linear ideal current sources").
* ``dense``    - incidence matrices A, A_s (Eqs. (4)-(5)), G, C, L, G_s, L_s
  (after Eq. (9)/(11)), system matrix M = C/h + G + hL (Eq. (11)), Lemma 1
  checks, direct (Cholesky) transient solves of Eq. (2), Eq. (10) and Eq. (11).
* ``nodal``    - the paper's nodal iteration in plain C (``nodal.c``): per-node
  update Eq. (12)-(13), SOR Eq. (15), Algorithm 1 time loop; companion
  (undifferenced, Eq. (10)) and second-order (Eq. (14)) right-hand sides.
* ``kcl``      - per-node Kirchhoff-current-law residual of a backward-Euler
  step (Eq. (12) discretised), the full-size parity property.

Pins: every function is checked by ``tests/test_oracle_*.py`` (-m "not gpu")
against closed forms, dense direct solves, invariants and the paper's stated
conditions; see DESIGN.md §4 for the pin table.  Functions without such a pin
are marked "parity unpinned" here and in DESIGN.md: (none at present).
"""
from . import netlist, pwl, dense, nodal, kcl  # noqa: F401
