"""CPU fp64 oracle for the RFDiffusion (RFD) graph-field integrator.

TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the C-ABI library
under ``paper_2302_00942_b200/`` and its Python binding) may import, call,
link or execute anything in this package.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs use it.

The oracle is written from the paper (arXiv 2302.00942, ``PAPER.md``) step by
step, in fp64, with no blocking, fusion or reordering beyond what the paper's
formulas state.  Every function cites the passage it follows.  Readings of
garbled or ambiguous passages are listed in ``DESIGN.md`` §3 (A1..A16) and
referenced here by their tag.

Modules
-------
philox  Philox4x32-10 counter-based generator (the random stream of a1).
rfd     frequencies, importance weights, features, Gram, core, integrate.
dense   exact epsilon-graph diffusion on tiny N (diagnostic, not a gate).

Pins (what each function is checked against, other than itself) are listed
in each module header and in ``DESIGN.md`` §4.  Functions without such a pin
say "parity unpinned".
"""
