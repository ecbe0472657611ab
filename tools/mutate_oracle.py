"""Mutation check of the oracle's SCG scalar logic (oracle/flmisr_oracle.c, orc_scg).

Each mutant changes ONE line of Moller's steps 3-8 (a dropped assignment, a flipped sign, a wrong
constant), is compiled to a temporary library, and the CPU pins are run against it through
ORACLE_LIB.  A mutant that no test kills is a hole in the pins.  Usage:

    python tools/mutate_oracle.py [--out profiles/r02_oracle_mutants.txt]
"""
from __future__ import annotations

import argparse
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "flmisr_oracle.c")

# (name, original text, mutated text) -- each original must occur exactly once in orc_scg
MUTANTS = [
    ("drop lamb<-lam on reject", "            lamb = lam;\n            success = 0;", "            success = 0;"),
    ("flip (1-Delta)", "lam = lam + delta * (1.0 - Delta) / pp;", "lam = lam + delta * (Delta - 1.0) / pp;"),
    ("recompute delta after reject", "            lamb = lam;\n            success = 0;", "            lamb = lam;"),
    ("repair: lamb sign", "lamb = 2.0 * (lam - delta / pp);", "lamb = 2.0 * (lam + delta / pp);"),
    ("repair: drop +lam pp", "delta = -delta + lam * pp;", "delta = -delta;"),
    ("repair: drop lam<-lamb", "                delta = -delta + lam * pp;\n                lam = lamb;",
     "                delta = -delta + lam * pp;"),
    ("drop PR+ clamp", "if (pr_plus && beta < 0.0) beta = 0.0;", ""),
    ("lam/4 -> lam/2", "lam = lam / 4.0;", "lam = lam / 2.0;"),
    ("delta scaling ignores lamb", "delta = delta + (lam - lamb) * pp;", "delta = delta + lam * pp;"),
    ("drop lamb<-0 on accept", "            lamb = 0.0;\n            success = 1;", "            success = 1;"),
    ("Delta without factor 2", "double Delta = 2.0 * delta * (f - fnew) / (mu * mu);",
     "double Delta = delta * (f - fnew) / (mu * mu);"),
    ("raise threshold 0.25 -> 0.75", "} else if (Delta < 0.25) {", "} else if (Delta < 0.75) {"),
    ("accept threshold 0 -> 0.25", "int acc = Delta >= 0.0;", "int acc = Delta >= 0.25;"),
    ("beta Fletcher-Reeves", "double beta = (rr - dot_consensus(pb, r, rold, g)) / mu;", "double beta = rr / mu;"),
    ("alpha sign", "double alpha = mu / delta;", "double alpha = -mu / delta;"),
]

TESTS = ["tests/test_oracle_scg_branches.py", "tests/test_oracle_pins.py"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    src = open(SRC).read()
    lines, survived = [], 0
    with tempfile.TemporaryDirectory() as td:
        for name, old, new in MUTANTS:
            assert src.count(old) == 1, (name, src.count(old))
            msrc = os.path.join(td, "m.c")
            mlib = os.path.join(td, f"m{len(lines)}.so")
            open(msrc, "w").write(src.replace(old, new))
            subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-o", mlib, msrc, "-lm"])
            env = dict(os.environ, ORACLE_LIB=mlib)
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "not gpu", "-p", "no:cacheprovider",
                                "-o", "addopts=", *TESTS], cwd=ROOT, env=env, capture_output=True, text=True)
            failed = [ln.split(" ")[1].split("::")[-1] for ln in r.stdout.splitlines() if ln.startswith("FAILED")]
            killed = r.returncode != 0
            survived += not killed
            lines.append(f"{'KILLED ' if killed else 'SURVIVED'} {name:32s} by {len(failed)} test(s): {', '.join(failed[:6])}")
            print(lines[-1], flush=True)
    summary = f"{len(MUTANTS) - survived}/{len(MUTANTS)} mutants killed"
    print(summary)
    if a.out:
        with open(a.out, "w") as f:
            f.write("# tools/mutate_oracle.py: one-line mutants of orc_scg (oracle/flmisr_oracle.c) vs the CPU pins\n")
            f.write("\n".join(lines) + "\n" + summary + "\n")
    return 1 if survived else 0


if __name__ == "__main__":
    sys.exit(main())
