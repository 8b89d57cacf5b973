"""Summarise a `-Xptxas -v` log (python paper_1810_11112_b200/_build.py
--ptxas-log=FILE): registers and spill bytes per kernel instantiation."""
import re
import subprocess
import sys


def parse(path):
    rows, cur = [], None
    for line in open(path):
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and cur:
            rows.append([cur, int(m.group(1)), int(m.group(2)), int(m.group(3)), None])
            continue
        m = re.search(r"Used (\d+) registers", line)
        if m and rows and rows[-1][0] == cur and rows[-1][4] is None:
            rows[-1][4] = int(m.group(1))
    names = subprocess.run(["cu++filt"], input="\n".join(r[0] for r in rows), capture_output=True,
                           text=True).stdout.splitlines()
    return [(n, *r[1:]) for n, r in zip(names, rows)]


if __name__ == "__main__":
    rows = parse(sys.argv[1])
    only_spills = "--spills" in sys.argv
    for name, stack, st, ld, regs in sorted(rows, key=lambda r: r[0]):
        if only_spills and not (st or ld):
            continue
        name = name.replace("cm::dev::", "").replace("(cm::dev::CollParams)", "")
        regs = "?" if regs is None else regs
        print(f"{regs:>4} regs {stack:>6} B stack {st:>6} B spill-st {ld:>6} B spill-ld  {name}")
    print(f"{len(rows)} kernels, {sum(1 for r in rows if r[2] or r[3])} with spills")
