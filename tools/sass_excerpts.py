"""Writes profiles/r02_sass_excerpts.txt: opcode counts and excerpts of the
hot loops from cuobjdump -sass of the built objects (no GPU needed)."""
import re
import subprocess
from collections import Counter


def sass(obj, fn):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    lines, on = [], False
    for ln in out.splitlines():
        if "Function :" in ln:
            on = fn in ln
        if on:
            lines.append(ln)
    return [re.sub(r"\s*/\* 0x[0-9a-f]+ \*/", "", ln) for ln in lines if ln.strip() and not re.match(r"^\s*/\* 0x", ln)]


def excerpt(rep, title, obj, fn, pat, ctx=6, maxn=1):
    L = sass(obj, fn)
    c = Counter()
    for ln in L:
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?P\d+\s+)?([A-Z0-9_.]+)", ln)
        if m:
            c[m.group(2)] += 1
    rep.append(f"==== {title}: {fn} ({obj}) - {len(L)} SASS lines")
    rep.append("opcode counts (top 18): " + ", ".join(f"{k} {v}" for k, v in c.most_common(18)))
    n = 0
    for i, ln in enumerate(L):
        if re.search(pat, ln):
            rep.append(f"-- excerpt around line {i}:")
            rep.extend(L[max(0, i - ctx):i + ctx + 1])
            n += 1
            if n >= maxn:
                break
    rep.append("")


if __name__ == "__main__":
    rep = []
    c = "paper_2412_12392_b200/csrc/"
    excerpt(rep, "matching refinement level 1 (exact int8 scores: IDP.4A = DP4A)", c + "match.o", "k_match_refine",
            r"IDP\.4A", ctx=10)
    excerpt(rep, "matching LM (256-bit ray-map gathers, FP64 interpolation)", c + "match.o", "k_match_refine",
            r"ENL2\.256", ctx=10)
    excerpt(rep, "backend edge terms (packed fp32 pairs: FFMA2 / FMUL2 / FADD2)", c + "backend.o",
            "k_edge_terms_ray", r"FFMA2", ctx=10)
    excerpt(rep, "backend edge terms (cp.async staging: LDGSTS)", c + "backend.o", "k_edge_terms_ray", r"LDGSTS", ctx=4)
    excerpt(rep, "frontal LDL^T solver", c + "backend.o", "k_ldlt_sky", r"MUFU\.RCP64H", ctx=6)
    excerpt(rep, "tracking GN (FP64 cost, packed fp32 sums)", c + "track.o", "k_track_gn", r"FFMA2|FMUL2", ctx=6)
    with open("profiles/r02_sass_excerpts.txt", "w") as f:
        f.write("# cuobjdump -sass excerpts of the hot loops (sm_100a), round 2 build\n"
                "# regenerate: python tools/sass_excerpts.py\n\n" + "\n".join(rep))
