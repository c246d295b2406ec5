"""Regenerate the closed-form golden fixtures (plain math only; imports neither
oracle/ nor the product)."""
import math
import os

HERE = os.path.dirname(os.path.abspath(__file__))


def write(name, header, rows):
    with open(os.path.join(HERE, name), "w") as f:
        for h in header:
            f.write(f"# {h}\n")
        for r in rows:
            f.write(" ".join(repr(float(x)) if not isinstance(x, int) else str(x) for x in r) + "\n")


def main():
    # ring C_n: lambda_m = 2 - 2 cos(2 pi m / n)  (BASELINE.json north_star; §2.1 L = S - W)
    for n in (8, 13):
        lam = sorted(2.0 - 2.0 * math.cos(2.0 * math.pi * m / n) for m in range(n))
        write(f"ring{n}_spectrum.txt",
              [f"Laplacian spectrum of the unit-weight ring C_{n}, ascending.",
               "Closed form lambda_m = 2 - 2 cos(2 pi m / n), m = 0..n-1 (circulant matrix).",
               "Cited by BASELINE.json north_star ('closed-form Laplacian spectra of ring and path graphs')."],
              [[x] for x in lam])
    # path P_n: lambda_m = 2 - 2 cos(pi m / n)
    for n in (3, 10):
        lam = sorted(2.0 - 2.0 * math.cos(math.pi * m / n) for m in range(n))
        write(f"path{n}_spectrum.txt",
              [f"Laplacian spectrum of the unit-weight path P_{n}, ascending.",
               "Closed form lambda_m = 2 - 2 cos(pi m / n), m = 0..n-1 (DCT-II eigenvectors)."],
              [[x] for x in lam])
    # Chebyshev coefficients of the ideal low-pass at lambda_c / lambda_max = 1/2:
    # x = 2 lambda/lambda_max - 1, cut at x = 0, theta_c = pi/2;
    # c_0 = 1/2, c_j = -2 sin(j pi / 2) / (pi j).
    rows = [[0, 0.5]] + [[j, -2.0 * math.sin(j * math.pi / 2.0) / (math.pi * j)] for j in range(1, 12)]
    write("cheb_step_half.txt",
          ["Chebyshev coefficients c_j of h(lambda) = 1[lambda <= lambda_max/2] on [0, lambda_max].",
           "PAPER.md Eq.(2) (l.126-130) ideal low-pass; Chebyshev basis per DESIGN.md R1.",
           "Closed form with theta_c = arccos(0) = pi/2: c_0 = 1 - theta_c/pi = 1/2,",
           "c_j = (2/pi) int_{theta_c}^{pi} cos(j t) dt = -2 sin(j pi/2)/(pi j).",
           "columns: j c_j"], rows)


if __name__ == "__main__":
    main()
