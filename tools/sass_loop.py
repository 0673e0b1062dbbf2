"""Print the instruction histogram (and optionally listing) of the hot sample loop of a kernel:
the backward-branch loop containing the most MUFU.EX2. Usage:
  python tools/sass_loop.py <obj-or-so> <function-substring> [--list]"""
import re
import subprocess
import sys
from collections import Counter


def functions(path):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    funcs, cur = {}, None
    for l in out.splitlines():
        m = re.search(r"Function : (\S+)", l)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m and cur:
            funcs[cur].append((int(m.group(1), 16), m.group(2).strip()))
    return funcs


def loops(ins):
    """All backward-branch loops with at least one EX2, as (ex2, body), innermost-first."""
    res = []
    for a, txt in ins:
        op = txt.split()[0] if not txt.startswith("@") else txt.split()[1]
        if op.startswith("BRA"):
            t = re.search(r"0x([0-9a-f]+)\s*$", txt)
            if t and int(t.group(1), 16) < a:
                lo = int(t.group(1), 16)
                body = [x for x in ins if lo <= x[0] <= a]
                ex2 = sum("MUFU.EX2" in x[1] for x in body)
                if ex2:
                    res.append((ex2, body))
    return sorted(res, key=lambda r: len(r[1]) / r[0])


def hot_loop(ins):
    best = None
    for a, txt in ins:
        op = txt.split()[0] if not txt.startswith("@") else txt.split()[1]
        if op.startswith("BRA"):
            t = re.search(r"0x([0-9a-f]+)\s*$", txt)
            if t and int(t.group(1), 16) < a:
                lo = int(t.group(1), 16)
                body = [x for x in ins if lo <= x[0] <= a]
                ex2 = sum("MUFU.EX2" in x[1] for x in body)
                if ex2 and (best is None or len(body) / ex2 < len(best[1]) / best[0]):
                    best = (ex2, body)
    return best


if __name__ == "__main__":
    import signal
    signal.signal(signal.SIGPIPE, signal.SIG_DFL)
    path, pat = sys.argv[1], sys.argv[2]
    for name, ins in functions(path).items():
        if pat not in name:
            continue
        which = int(sys.argv[sys.argv.index("--loop") + 1]) if "--loop" in sys.argv else 0
        ex2, body = loops(ins)[which]
        ops = Counter((t.split()[1] if t.startswith("@") else t.split()[0]) for _, t in body)
        print(f"{name}\n  loop: {len(body)} instructions, {ex2} EX2 -> {len(body)/max(ex2,1):.1f} per sample")
        for op, c in ops.most_common():
            print(f"    {c:4d} {op}")
        if "--list" in sys.argv:
            for a, t in body:
                print(f"    {a:05x}  {t}")
