#!/usr/bin/env python
"""profiles/r02_sass_k_brick2_p5.txt: opcode histogram and the async-copy / barrier / register re-allocation
instructions of k_brick2<5,double> from the built object (cuobjdump -sass)."""
import collections, re, subprocess
obj = "paper_2205_08909_b200/csrc/build/mfcg_inst_p5.o"
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout.splitlines()
ins, on = [], False
for l in out:
    if "Function :" in l:
        on = "k_brick2ILi5Ed" in l
    m = re.match(r"\s+/\*([0-9a-f]{4,6})\*/\s+(.*?);", l)
    if on and m:
        ins.append((m.group(1), re.sub(r"\s+", " ", m.group(2)).strip() + " ;"))
def opcode(t):
    t = t.split()
    return t[1] if t[0].startswith("@") else t[0]
hist = collections.Counter(opcode(t) for _, t in ins)
keys = ("UBLKCP", "SYNCS", "USETMAXREG", "LDGSTS", "LDGDEPBAR", "DEPBAR", "FENCE", "ARRIVES", "BAR.", "LDL", "STL", "RED.", "STG.E.128", "LDS.128")
sel = [(a, t) for a, t in ins if any(k in t for k in keys)]
with open("profiles/r02_sass_k_brick2_p5.txt", "w") as f:
    f.write(f"# SASS of k_brick2<5,double> (cuobjdump -sass {obj}), round 2, final build; tools/sass_listing2.py\n"
            "# TMA-class bulk copies: UBLKCP.S.G (cp.async.bulk global -> shared, mbarrier complete_tx); SYNCS.* = mbarrier\n"
            "# arrive / expect_tx / try_wait; USETMAXREG = setmaxnreg register re-allocation between the warpgroups;\n"
            "# LDGSTS = cp.async of the brick-boundary values; 128-bit shared loads / global stores in the update warps;\n"
            f"# LDL / STL (spills): {sum(v for k, v in hist.items() if k.startswith(('LDL', 'STL')))}.\n"
            f"# {len(ins)} instructions; opcode histogram (top 40):\n")
    for k, v in hist.most_common(40):
        f.write(f"#   {k} {v}\n")
    f.write("# selected instructions (address  instruction):\n")
    for a, t in sel:
        f.write(f"{a}  {t}\n")
print(len(ins), "instructions;", {k: sum(1 for _, t in ins if k in t) for k in ("UBLKCP", "USETMAXREG", "LDGSTS", "LDL", "STL")})
