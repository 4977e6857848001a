"""Small end-to-end run for compute-sanitizer (racecheck / synccheck /
memcheck, one tool per call): C1-like 2D Laplacian (n = 1024, L5) with a
multi-CTA RRQR group, factorize + PCG, checked against the oracle."""
import sys
sys.path.insert(0, '.')
import __graft_entry__ as g
g.smoke()
