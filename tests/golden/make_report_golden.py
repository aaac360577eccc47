"""Generate the wire-format fixtures under tests/golden/report/ with the
REFERENCE's own writers (tpfem/report.hpp via oracle/report_fixture.cpp).

TEST INFRASTRUCTURE: run here (needs /root/reference and `make -C oracle
report-fixture`); the outputs are committed and the tests only read them.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
OUT = os.path.join(HERE, "report")
BIN = os.path.join(ROOT, "oracle", "_ref", "report_fixture")

# synthetic SolveReports covering: tiny/huge/denormal magnitudes, exact
# integers, negative exponents, NaN q (omitted), several methods and statuses
SPEC = """m1 converged 4 0.123456789 0.3333333333333333 5 1.0 0.5 0.0625 1e-05 3.3e-09 4 0.5 0.125 0.00016 0.00033
m2 max_iter 3 12.5 nan 4 65312.4 1.5e+300 2.2250738585072014e-308 7.0 3 2.0 1.0000000000000002 -0.0
m3 stalled 0 0.0 0.95 9 6.02214076e+23 1e+15 999999999999999.9 1234567890123456.0 0.0001 0.00012345 100.0 -3.5 5e-324 0
T 16 306 0.001953125 9 0.25 3 1.75 0 0.0
T 256 65025 0.1 165 1.2339222402572632 0 0.0 7 3e-05
"""


def main():
    if not os.path.exists(BIN):
        subprocess.check_call(["make", "-C", os.path.join(ROOT, "oracle"), "report-fixture"])
    os.makedirs(OUT, exist_ok=True)
    spec = os.path.join(OUT, "spec.txt")
    with open(spec, "w") as f:
        f.write(SPEC)
    subprocess.check_call([BIN, spec, OUT])
    subprocess.check_call([BIN, "vtk", OUT])  # mesh.vtk, u.vtk (vtk.hpp)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    sys.exit(main())
