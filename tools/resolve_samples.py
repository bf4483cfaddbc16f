"""Symbolise SPQR_SAMPLE output locally: self and inclusive sample counts per function."""
import collections
import subprocess
import sys

path = sys.argv[1]
lib = sys.argv[2] if len(sys.argv) > 2 else "paper_2102_09878_b200/libspaqr_b200.so"
stacks = []
offs = set()
for line in open(path):
    frames = []
    for fr in line.strip().split(" | "):
        if not fr:
            continue
        obj, _, off = fr.rpartition(" ")
        frames.append((obj, int(off)))
        if obj.endswith("libspaqr_b200.so"):
            offs.add(int(off))
    stacks.append(frames)
offs = sorted(offs)
names = {}
if offs:
    out = subprocess.run(["addr2line", "-f", "-C", "-e", lib] + [hex(o - 1) for o in offs], capture_output=True,
                         text=True).stdout.splitlines()
    for i, o in enumerate(offs):
        fn = out[2 * i] if 2 * i < len(out) else "?"
        fn = fn.replace("(anonymous namespace)", "anon")
        names[o] = fn.split("(")[0][-90:]
import bisect, os
symtabs = {}
def dyn_name(obj, off):
    if obj not in symtabs:
        syms = []
        if os.path.exists(obj):
            out = subprocess.run(["nm", "-D", "--defined-only", obj], capture_output=True, text=True).stdout
            for l in out.splitlines():
                p = l.split()
                if len(p) >= 3:
                    try:
                        syms.append((int(p[0], 16), p[2]))
                    except ValueError:
                        pass
        syms.sort()
        symtabs[obj] = syms
    syms = symtabs[obj]
    i = bisect.bisect_right(syms, (off, "~")) - 1
    base = obj.split("/")[-1]
    return f"{base}:{syms[i][1]}" if i >= 0 else base
self_c = collections.Counter()
incl = collections.Counter()
for st in stacks:
    seen = set()
    for k, (obj, off) in enumerate(st):
        nm = names.get(off, obj.split("/")[-1]) if obj.endswith("libspaqr_b200.so") else dyn_name(obj, off)
        if k == 0:
            self_c[nm] += 1
        if nm not in seen:
            incl[nm] += 1
            seen.add(nm)
n = len(stacks)
print(f"{n} samples")
print("--- self")
for nm, c in self_c.most_common(30):
    print(f"{100*c/n:6.1f}%  {nm}")
print("--- inclusive")
for nm, c in incl.most_common(40):
    print(f"{100*c/n:6.1f}%  {nm}")
# SAMPLE_FOCUS=<substring>: for samples whose leaf frames (first 6) match it, the nearest
# libspaqr_b200.so frame — which engine code pays for it
focus = os.environ.get("SAMPLE_FOCUS")
if focus:
    by = collections.Counter()
    for st in stacks:
        nm0 = [names.get(off, obj.split("/")[-1]) if obj.endswith("libspaqr_b200.so") else dyn_name(obj, off)
               for obj, off in st]
        if not any(focus in x for x in nm0[:6]):
            continue
        own = [x for (obj, _), x in zip(st, nm0) if obj.endswith("libspaqr_b200.so")]
        by[" < ".join(own[:3]) if own else "?"] += 1
    print(f"--- '{focus}' by engine caller")
    for nm, c in by.most_common(25):
        print(f"{100*c/n:6.1f}%  {nm}")
