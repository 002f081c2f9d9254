"""One-off authoring script: copy the numbers PAPER.md prints in its figure sources into
tests/golden/ with line citations.  Run once when authoring; tests read only tests/golden/.
Usage: python tools/extract_golden.py /root/reference/PAPER.md
"""
import re
import sys

paper = open(sys.argv[1]).read().splitlines()


def rows(start, end):
    out = []
    for ln in range(start, end + 1):
        m = re.match(r"^\s*([0-9.eE+-]+)\s+([0-9.eE+-]+)\\\\", paper[ln - 1])
        if m:
            out.append((ln, m.group(1), m.group(2)))
    return out


def dump(path, header, data):
    with open(path, "w") as fh:
        for h in header:
            fh.write("# " + h + "\n")
        for ln, a, b in data:
            fh.write(f"{a} {b}  # P:{ln}\n")


dump("tests/golden/fig4a_karate_L_true.txt",
     ["PAPER.md Fig. 4(a) 'True value' curve (P:1223-1256): average return probability",
      "(eq:average_return_probabilities) of the standard Laplacian L on Newman/karate.",
      "columns: t  p_hat(t)"], rows(1224, 1255))
dump("tests/golden/fig4b_karate_nbt_resolvent_true.txt",
     ["PAPER.md Fig. 4(b) 'True value' curve (P:1426-1459): average return probability of",
      "L_1((1-alpha x)^{-1}), alpha = 1/(1+rho(Z)) (caption P:1260) on Newman/karate.",
      "columns: t  p_hat(t)"], rows(1427, 1458))
panels = {"L": 762, "res": 803, "exp": 844, "nbt_exp": 926}
with open("tests/golden/fig1_g58_stationary.txt", "w") as fh:
    fh.write("# PAPER.md Fig. 1 (P:695-950): stationary distribution of the Markov chain induced by\n")
    fh.write("# each Laplacian on the trap graph G_{5,8} (P:663-690); paper node labels 1..13.\n")
    fh.write("# panels: L (standard), res = L((1-alpha x)^-1) alpha=1/(2 rho(A)) (caption P:947),\n")
    fh.write("# exp = L(exp), nbt_exp = L_1(exp).  (The k-path panel is out of scope.)\n")
    fh.write("# columns: panel node value\n")
    for name, start in panels.items():
        for ln, node, val in rows(start, start + 20):
            fh.write(f"{name} {node} {val}  # P:{ln}\n")
print("ok")
