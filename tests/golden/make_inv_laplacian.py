"""Writes tests/golden/inv_laplacian_n8.txt: exact y = A x for the inverse 1D
Laplacian A = tridiag(-1,2,-1)^{-1} (BASELINE.json config 5's closed form
A_ij = min(i,j)(n+1-max(i,j))/(n+1); eq. (8) P:1314-1322 up to -1/h^2), n = 8,
x in {[1,-2,3,-4,5,-6,7,-8], [3,1,4,1,5,9,2,6]}. Exact rational arithmetic (fractions); it asserts
T A = I exactly before writing. Calls nothing from the CUDA path or oracle/."""
from fractions import Fraction
import os

n = 8
A = [[Fraction(min(i, j) * (n + 1 - max(i, j)), n + 1) for j in range(1, n + 1)] for i in range(1, n + 1)]
T = [[(2 if i == j else (-1 if abs(i - j) == 1 else 0)) for j in range(n)] for i in range(n)]
for i in range(n):
    for j in range(n):
        assert sum(T[i][t] * A[t][j] for t in range(n)) == (1 if i == j else 0)
xs = [[1, -2, 3, -4, 5, -6, 7, -8], [3, 1, 4, 1, 5, 9, 2, 6]]
ys = [[sum(A[i][j] * x[j] for j in range(n)) for i in range(n)] for x in xs]
out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "inv_laplacian_n8.txt")
with open(out, "w") as f:
    f.write("# Exact y = A x, A = tridiag(-1,2,-1)^{-1}, n = 8 (closed form of BASELINE config 5;\n")
    f.write("# eq. (8) P:1314-1322). Written by tests/golden/make_inv_laplacian.py (exact rationals).\n")
    for x, y in zip(xs, ys):
        f.write("x: " + " ".join(str(v) for v in x) + "\n")
        f.write("y: " + " ".join(f"{v.numerator}/{v.denominator}" for v in y) + "\n")
