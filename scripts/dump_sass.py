"""Write the SASS of every kernel instantiation the bench times to profiles/sass/
(cuobjdump of the exact libdpdb.so the bench loads), plus an index with the
library's sha256 and per-kernel instruction counts.

    python scripts/dump_sass.py
"""
import hashlib
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1311_0402_b200", "libdpdb.so")
OUT = os.path.join(ROOT, "profiles", "sass")
# file name -> mangled symbol (the C3 step loop's launches; pack/unpack: brick halo)
KERNELS = {
    "force_walk_fuse_streams": "_ZN4dpdb12k_force_walkILb0ELb0ELi128ELi1EEEvNS_9ForceArgsE",
    "force_walk_fuse_keys": "_ZN4dpdb12k_force_walkILb0ELb0ELi128ELi2EEEvNS_9ForceArgsE",
    "force_walk_nofuse": "_ZN4dpdb12k_force_walkILb0ELb0ELi128ELi0EEEvNS_9ForceArgsE",
    "build_range_walk": "_ZN4dpdb13k_build_rangeILb1ELb0EEEvNS_9BuildArgsE",
    "onesweep_hist": "_ZN4dpdb15k_onesweep_histEPKjjiPj",
    "onesweep": "_ZN4dpdb10k_onesweepEPKjS1_PjS2_jijS1_S2_S2_",
    "permute": "_ZN4dpdb9k_permuteILb0ELb0EEEvNS_11PermuteArgsE",
    "integrate_final": "_ZN4dpdb11k_integrateILb1ELb0ELb0ELb0EEEvNS_13IntegrateArgsE",
    "pack_update": "_ZN4dpdb6k_packILb1EEEvNS_8PackArgsEPv",
    "unpack_update": "_ZN4dpdb8k_unpackILb1EEEvNS_10UnpackArgsEPKv",
    "put_ghost_update": "_ZN4dpdb5k_putENS_7PutArgsE",
}


def main():
    sha = hashlib.sha256(open(LIB, "rb").read()).hexdigest()
    full = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    funcs = {}
    cur = None
    for line in full.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = [line.strip()]
        elif cur:
            funcs[cur].append(line)
    for f in os.listdir(OUT):
        if f.endswith(".sass"):
            os.remove(os.path.join(OUT, f))
    rows = []
    for name, sym in KERNELS.items():
        body = funcs[sym]
        ins = [l for l in body if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l)]
        ops = [re.sub(r"^\s*/\*[0-9a-f]+\*/\s*(@!?U?P\w+\s+)?", "", l).split()[0] for l in ins if l.strip()]
        hist = {k: sum(1 for o in ops if o.startswith(k)) for k in
                ("LDG", "STG", "LDS", "STS", "ATOMS", "REDG", "ATOMG", "MUFU", "DADD", "DFMA", "DMUL", "VOTE",
                 "BAR", "UTMALDG", "UBLKCP", "LDGSTS")}
        with open(os.path.join(OUT, name + ".sass"), "w") as fh:
            fh.write(f"# cuobjdump -sass paper_1311_0402_b200/libdpdb.so (sm_100a, sha256 {sha[:16]}), {sym}\n")
            fh.write("\n".join(body) + "\n")
        rows.append((name, sym, len(ops), hist))
    with open(os.path.join(OUT, "INDEX.md"), "w") as fh:
        fh.write(f"# SASS listings of `paper_1311_0402_b200/libdpdb.so` (sha256 `{sha}`)\n\n")
        fh.write("Written by `python scripts/dump_sass.py` from the library the bench and tests load.\n\n")
        keys = list(rows[0][3])
        fh.write("| file | kernel | instructions | " + " | ".join(keys) + " |\n")
        fh.write("|---|---|---|" + "---|" * len(keys) + "\n")
        for name, sym, n, h in rows:
            fh.write(f"| `{name}.sass` | `{sym}` | {n} | " + " | ".join(str(h[k]) for k in keys) + " |\n")
    print(open(os.path.join(OUT, "INDEX.md")).read())


if __name__ == "__main__":
    main()
