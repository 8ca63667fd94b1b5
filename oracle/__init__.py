"""CPU oracle for arXiv 1606.05562 (16-point multiplierless approximate DCT).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import, call or
execute anything under ``oracle/``.  The product path (``paper_1606_05562_b200``
and its CUDA library) never imports this package and this package never imports
the product path: the two share no code, no constants and no helpers.  Inputs
come from the neutral generator module ``synth`` which holds none of the
method's arithmetic.

Every function is a plain, slow, obviously-correct restatement of the paper
(PAPER.md line numbers are cited per function), evaluated in float64 or exact
integers.  Where the paper is silent or garbled the readings of DESIGN.md §3
(IDs A1..A20, taken from SURVEY.md §8(c)) are used and cited.

Pins (what this oracle is checked against, other than itself) live in
``tests/test_oracle_pins.py``; the only function without an external pin is
listed in DESIGN.md §3 as "parity unpinned" (the exact-DCT APE comparison of
config 5 against the paper's Lena / USC-SIPI figures, whose images are absent).
"""
