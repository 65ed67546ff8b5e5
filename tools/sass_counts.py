"""Static SASS opcode counts of the product kernels (cuobjdump -sass of the
build objects): the evidence that the tcgen05 path issues UTCHMMA / LDTM /
UTCBAR and the team kernel FFMA2 (development aid; output kept in profiles/)."""
import re, subprocess, sys
from collections import Counter

OPS = ["UTCHMMA", "UTCBAR", "LDTM", "STTM", "SYNCS", "UTMALDG", "FFMA2", "FMUL2", "FADD2", "FFMA", "FMUL", "FADD",
       "LDS", "STS", "SHFL", "BAR", "LDG", "STG", "LDL", "STL"]


def counts(obj):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    res, fn = {}, None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            fn = m.group(1)
            res[fn] = Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
        if m and fn:
            res[fn][m.group(1)] += 1
            res[fn]["_total"] += 1
    return res


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    return dict(zip(names, r))


if __name__ == "__main__":
    for obj in sys.argv[1:]:
        res = counts(obj)
        dm = demangle(list(res))
        print(f"== {obj}")
        for fn, c in res.items():
            name = re.sub(r"ufpgd_gpu_impl::\(anonymous namespace\)::", "", dm[fn])
            name = re.sub(r"\(ufpgd_gpu_impl::FusedArgs.*", "", name)
            if not any(c[o] for o in ("UTCHMMA", "FFMA2")):
                continue
            print(f"{name[:110]}")
            print("   total " + str(c["_total"]) + "  " + "  ".join(f"{o} {c[o]}" for o in OPS if c[o]))
