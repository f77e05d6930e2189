#!/usr/bin/env python
"""Mutation check of the oracle's CPU pins (no GPU).

Copies the repo's oracle + tests to a scratch directory, applies one
plausible mistake at a time to oracle/oracle.cpp (a dropped term, a wrong
comparison, a flipped tie-break, a broken counter ...), rebuilds the oracle
and runs the `-m "not gpu"` oracle pins.  Every mutation must make at least
one pin fail; the script prints one line per mutation and exits 1 if any
survives.  Usage: python tools/oracle_mutations.py
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (description, exact text in oracle.cpp, replacement)
MUTATIONS = [
    ("R13: drop the 'Evaluate changed nothing' clause",
     "if (!ptr_changed && !changed)", "if (!ptr_changed)"),
    ("R13: drop the 'no parent change' clause",
     "if (!ptr_changed && !changed)", "if (!changed)"),
    ("relaxation counter counts vertices, not edges",
     "relax += (int64_t)c->in[v].size();", "relax += 1;"),
    ("visit counter double counts", "++visits;", "visits += 2;"),
    ("epsilon ignored (R5)", "if (dg <= c->epsilon) break;", "if (dg <= 0.0) break;"),
    ("strict < becomes <= in Improve (P:246)", "if (best < c->g[v]) {  // strict", "if (best <= c->g[v]) {  // strict"),
    ("tie-break on the highest id (R6)",
     "if (cand < best || (cand == best && arg >= 0 && uc.first < arg)) {",
     "if (cand < best || (cand == best && arg >= 0 && uc.first > arg)) {"),
    ("Evaluate without the B reset (P:256)",
     "std::fill(c->b.begin(), c->b.end(), 0);  // B <- {} (P:256)", ""),
    ("child test with <= (P:263)", ": (c->g[v] + c->h[v] < thr);", ": (c->g[v] + c->h[v] <= thr);"),
    ("Delta g as the last vertex's delta (R1 literal)", "if (d > dg) dg = d;", "dg = d;"),
    ("goal not always improved (R4)",
     "if (!(prune_off || c->b[v] || is_goal(c, v) || (!nbr.empty() && nbr[v]))) continue;",
     "if (!(prune_off || c->b[v] || (!nbr.empty() && nbr[v]))) continue;"),
    ("NEIGHBOURS: the root is not a source (R16)",
     "if (uc.first == kRoot || c->b[uc.first]) { nbr[v] = 1; break; }",
     "if (c->b[uc.first]) { nbr[v] = 1; break; }"),
    ("NEIGHBOURS: only the root is a source (R16)",
     "if (uc.first == kRoot || c->b[uc.first]) { nbr[v] = 1; break; }",
     "if (uc.first == kRoot) { nbr[v] = 1; break; }"),
    ("NEIGHBOURS: neighbours never join I (R16)",
     "if (!(prune_off || c->b[v] || is_goal(c, v) || (!nbr.empty() && nbr[v]))) continue;",
     "if (!(prune_off || c->b[v] || is_goal(c, v))) continue;"),
    ("local relaxation keeps the highest id on ties (R14, R6)",
     "if (cand < best || (cand == best && arg >= 0 && u < arg)) {",
     "if (cand < best || (cand == best && arg >= 0 && u > arg)) {"),
    ("new vertex promising test with <= (P:186-187)",
     "c->b[v] = (c->g[v] + c->h[v] < thr) ? 1 : 0;", "c->b[v] = (c->g[v] + c->h[v] <= thr) ? 1 : 0;"),
    ("Evaluate adds the parent's cost instead of the child's (R9)",
     "c->g[v] = c->g[p] + c->pc[v];  // g(n) <- c(v,n) + g(v), P:262",
     "c->g[v] = c->g[p] + c->pc[p];  // g(n) <- c(v,n) + g(v), P:262"),
]

PIN_TESTS = ["tests/test_oracle_loop_pins.py", "tests/test_oracle_pins.py",
             "tests/test_oracle_goals_variants.py", "tests/test_oracle_neighbours.py"]


def main():
    src = open(os.path.join(ROOT, "oracle", "oracle.cpp")).read()
    survivors = 0
    with tempfile.TemporaryDirectory() as tmp:
        for d in ("oracle", "gen", "tests", "paper_2003_04920_b200"):
            shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                            ignore=shutil.ignore_patterns("*.cu", "*.cuh", "lib"))
        shutil.copy(os.path.join(ROOT, "pytest.ini"), tmp)
        for desc, old, new in MUTATIONS:
            if old not in src:
                print(f"MISSING  {desc}: pattern not found")
                survivors += 1
                continue
            with open(os.path.join(tmp, "oracle", "oracle.cpp"), "w") as f:
                f.write(src.replace(old, new, 1))
            subprocess.run(["g++", "-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-shared",
                            "-o", os.path.join(tmp, "oracle", "liboracle.so"),
                            os.path.join(tmp, "oracle", "oracle.cpp")], check=True)
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "not gpu", "-x",
                                "-p", "no:cacheprovider"] + PIN_TESTS, cwd=tmp,
                               capture_output=True, text=True)
            killed = r.returncode != 0
            survivors += 0 if killed else 1
            print(f"{'killed ' if killed else 'SURVIVED'} {desc}: {r.stdout.strip().splitlines()[-1]}")
    sys.exit(1 if survivors else 0)


if __name__ == "__main__":
    main()
