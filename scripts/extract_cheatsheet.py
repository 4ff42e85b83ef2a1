"""Dev-time extractor: writes tests/golden/faa_di_bruno_nu.txt from the paper's
Faa di Bruno cheat sheet (App. A), h-column only.

Each line of the fixture: k, the partition (parts, non-increasing), nu, and the
PAPER.md line it was read from. The trivial partition {k} (the term
<dh, x_k>, coefficient 1) is included. Run once; the fixture is committed.
"""
import re
import sys

src = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/PAPER.md"
lines = open(src).read().split("\n")
out = []
k = None
term = re.compile(r"^\s*(\+\s*)?(\d+)?\s*\\langle \\partial(\^\{(\d+)\})? \{\\bm\{h\}\}, (.*)\\rangle")
for i in range(1269, 1965):
    s = lines[i]
    m = re.search(r"\{\\bm\{h\}\}_\{(\d+)\}$", s.strip())
    if m and "=" not in s:
        k = int(m.group(1))
        continue
    m = term.match(s)
    if not m or k is None:
        continue
    coef = int(m.group(2)) if m.group(2) else 1
    order = int(m.group(4)) if m.group(4) else 1
    parts = []
    for idx, pw in re.findall(r"\{\\bm\{x\}\}_\{(\d+)\}(?:\^\{\\otimes(\d+)\})?", m.group(5)):
        parts += [int(idx)] * (int(pw) if pw else 1)
    assert len(parts) == order and sum(parts) == k, (i + 1, s)
    out.append((k, tuple(sorted(parts, reverse=True)), coef, i + 1))
with open("tests/golden/faa_di_bruno_nu.txt", "w") as fh:
    fh.write("# Faa di Bruno multiplicities nu(sigma), Eq. 3 (P:386-415), read from the\n")
    fh.write("# cheat sheet of App. A (PAPER.md P:1270-1965), h-column. Format:\n")
    fh.write("# k | parts (non-increasing) | nu | PAPER.md line\n")
    for k_, parts, coef, ln in out:
        fh.write(f"{k_} | {' '.join(map(str, parts))} | {coef} | P:{ln}\n")
print(len(out), "terms")
