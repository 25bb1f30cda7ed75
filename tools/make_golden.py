"""Write tests/golden/omega_seed1_800x25.txt: sampled Ω entries for seed=1, n=800, ℓ=25
(config C1's Ω).  Calls only oracle/ (regression fixture; the pins are in test_oracle_pins)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

Om = oracle.omega(1, 800, 25)
idx = [(0, 0), (1, 0), (2, 0), (3, 0), (799, 0), (0, 1), (123, 7), (799, 24), (400, 12), (5, 24)]
with open(os.path.join(ROOT, "tests", "golden", "omega_seed1_800x25.txt"), "w") as f:
    f.write("# Ω(i,j) for seed=1, n=800, l=25 (DESIGN.md §4 RNG layout); written by tools/make_golden.py\n")
    for i, j in idx:
        f.write(f"{i} {j} {float(Om[i, j])!r}\n")
