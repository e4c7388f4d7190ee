"""TEST-INPUT GENERATOR: writes contracts/worst-off.cl and contracts/brc.cl.

The worst-off autocallable and the barrier reverse convertible named by
BASELINE.json do not ship with the reference; they are authored in the
reference's own contract language (CL, proj/src/parser.cpp) exactly as
SURVEY.md Appendix A specifies, and compiled by the reference itself
(oracle/make_golden.py) into the kernels the GPU engine prices.
"""
import os

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "..", "contracts")


def worst() -> str:
    a = "obs(SX5E,0)/3758.05"
    b = "obs(N225,0)/11840.0"
    c = "obs(SPX,0)/1200.0"
    return f"cond({a} < {b}, cond({a} < {c}, {a}, {c}), cond({b} < {c}, {b}, {c}))"


def worst_off_cl() -> str:
    w = worst()
    c = (f"translate(73, scale(cond(1.0 <= {w}, 1750.0, cond(0.75 < {w}, 1000.0, "
         f"1000.0 * {w})), transfer(you, me, EUR)))")
    for amt in reversed([1150.0, 1300.0, 1450.0, 1600.0]):
        c = f"translate(73, if(1.0 <= {w}, scale({amt}, transfer(you, me, EUR)), {c}))"
    return "-- worst-off autocallable, 3 underlyings x 5 dates\n" + c + "\n"


def brc_cl() -> str:
    w = worst()
    hit = " | ".join(f"obs(SX5E,{-k}) <= 2630.635 | obs(N225,{-k}) <= 8288.0 | obs(SPX,{-k}) <= 840.0"
                     for k in range(366, -1, -1))
    below = "obs(SX5E,0) < 3758.05 | obs(N225,0) < 11840.0 | obs(SPX,0) < 1200.0"
    return ("-- barrier reverse convertible, 3 underlyings x 367 dates\n"
            f"both(scale(100.0, translate(366, transfer(you, me, EUR))),\n"
            f" translate(366, if(({below}) & ({hit}),\n"
            f"   scale(1000.0 * {w}, transfer(you, me, EUR)),\n"
            f"   scale(1000.0, transfer(you, me, EUR)))))\n")


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, "worst-off.cl"), "w") as f:
        f.write(worst_off_cl())
    with open(os.path.join(OUT, "brc.cl"), "w") as f:
        f.write(brc_cl())
