"""List each global load in a kernel's SASS and the first later instruction
that reads its destination register (distance in instructions): a short
distance means the load latency is exposed.  usage: sass_ldg_uses.py obj kernel_substr"""
import re, subprocess, sys
obj, kname = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
for f in funcs:
    head = f.split("\n", 1)[0]
    if kname not in head:
        continue
    print("==", head)
    ins = []
    for line in f.split("\n"):
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((m.group(1), m.group(2).strip()))
    for k, (addr, txt) in enumerate(ins):
        if re.search(r"\b(LDG|LDL|LD)\.", txt):
            m = re.search(r"(LDG|LDL|LD)\S*\s+(R\d+)", txt)
            if not m:
                continue
            reg = m.group(2)
            rn = int(reg[1:])
            opc = txt.split()[0] if not txt.startswith("@") else txt.split()[1]
            wide = opc.endswith((".64", ".128"))
            regs = {f"R{rn}"} | ({f"R{rn+1}"} if wide else set())
            use = None
            for j in range(k + 1, min(k + 400, len(ins))):
                t = ins[j][1]
                ops = t.split(None, 1)
                if len(ops) < 2:
                    continue
                srcs = ops[1].split(",", 1)
                src = srcs[1] if len(srcs) > 1 and not ops[0].startswith(("ST", "RED", "ATOM")) else ops[1]
                if any(re.search(rf"\b{r}\b", src) for r in regs):
                    use = (j - k, t)
                    break
            print(f"{addr}: {txt[:70]:70s} -> +{use[0] if use else '-'}: {use[1][:60] if use else ''}")
