"""Report the hot inner loop of a kernel in libebc200.so: size, FFMA/FADD count,
FFMA register-bank parity conflicts (after operand reuse)."""
import re, subprocess, sys
pat = sys.argv[1]
lib = sys.argv[2] if len(sys.argv) > 2 else "paper_2105_12026_b200/libebc200.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
for f in funcs:
    name = f.split("\n", 1)[0]
    if not re.search(pat, name):
        continue
    ins = []
    for l in f.splitlines():
        m = re.search(r"/\*([0-9a-f]{4,5})\*/\s+(.*?);", l)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    best = None
    for a, t in ins:
        m = re.search(r"BRA(?:\.U)? (?:!?U?P\d, )?(0x[0-9a-f]+)", t)
        if m and int(m.group(1), 16) < a:
            tgt = int(m.group(1), 16)
            body = [x for x in ins if tgt <= x[0] <= a]
            nf = sum(1 for x in body if x[1].startswith(("FFMA", "FADD")))
            if best is None or nf > best[1] or (nf == best[1] and len(body) < len(best[0])):
                best = (body, nf)
    if not best:
        continue
    body, nf = best
    conf = 0
    for _, t in body:
        m = re.match(r"FFMA R(\d+), R(\d+)(\.reuse)?, R(\d+)(\.reuse)?, R(\d+)(\.reuse)?", t)
        if not m:
            continue
        regs = [(int(m.group(2)), bool(m.group(3))), (int(m.group(4)), bool(m.group(5))), (int(m.group(6)), bool(m.group(7)))]
        srcs = set(r for r, f in regs if not f)
        ev = len([x for x in srcs if x % 2 == 0])
        if max(ev, len(srcs) - ev) > 1:
            conf += 1
    others = {}
    for _, t in body:
        op = t.split()[0]
        if not op.startswith(("FFMA", "FADD")):
            others[op] = others.get(op, 0) + 1
    print(f"{name[:110]}\n  loop {len(body)} instr, {nf} FFMA/FADD ({nf/len(body):.3f}), FFMA bank conflicts {conf}, other {others}")
