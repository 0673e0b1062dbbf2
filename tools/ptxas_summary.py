import re, sys
lines = sys.stdin.read().splitlines()
cur = None
for i, l in enumerate(lines):
    m = re.search(r"Compiling entry function '(\S+)'", l)
    if m:
        cur = m.group(1); continue
    if cur and 'registers' in l:
        name = cur
        mm = re.search(r'solve_kernelINS_\d+(\w+?)ILi(\d+)', name)
        if mm: name = f"solve {mm.group(1)} n={mm.group(2)}"
        else: name = name[:60]
        st = lines[i-1].strip()
        print(f"{name:40s} {l.split('Used')[1].split(',')[0].strip():16s} | {st}")
        cur = None
