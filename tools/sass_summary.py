"""profiles/r2_sass_summary.md: ptxas register / spill figures and SASS opcode
histograms of the step kernels of the in-tree libmlob.so (dev tool).
  python tools/sass_summary.py"""
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KERNELS = {
    "_ZN4mlob11book_kernelILi4ELb0ELb1EEEvNS_7KParamsE": "book_kernel<4, false, true> (C <= 128, register book, large batches)",
    "_ZN4mlob11book_kernelILi32ELb0ELb0EEEvNS_7KParamsE": "book_kernel<32, false, false> (C <= 1024, shared-memory book)",
    "_ZN4mlob10act_kernelENS_7KParamsE": "act_kernel",
    "_ZN4mlob14outcome_kernelENS_7KParamsE": "outcome_kernel",
    "_ZN4mlob12reset_kernelENS_7KParamsE": "reset_kernel",
}
KEY = ("UBLKCP", "SYNCS", "CREDUX", "REDUX", "VOTE", "UTMA", "LDL", "STL", "BAR", "WARPSYNC")


def main():
    tmp = "/tmp/mlob_cubins"
    subprocess.run(f"rm -rf {tmp} && mkdir -p {tmp} && cd {tmp} && cuobjdump -xelf all "
                   f"{ROOT}/paper_2511_02136_b200/libmlob.so > /dev/null", shell=True, check=True)
    sass = subprocess.run(f"cuobjdump -sass {tmp}/mlob_kernels.sm_100a.cubin", shell=True, capture_output=True,
                          text=True).stdout
    funcs, cur = {}, None
    for ln in sass.split("\n"):
        m = re.search(r"Function : (\S+)", ln)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,6}\*/\s+(@!?U?P[T0-9]+\s+)?([A-Z][A-Z0-9_.]*)", ln)
        if m and cur:
            funcs[cur].append(m.group(2))
    ptx = subprocess.run("nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 --fmad=false -Xptxas -v "
                         "-c -o /dev/null csrc/mlob_kernels.cu", shell=True, capture_output=True, text=True,
                         cwd=os.path.join(ROOT, "paper_2511_02136_b200")).stderr.split("\n")
    info = {}
    for i, ln in enumerate(ptx):
        m = re.search(r"Compiling entry function '(\S+)'", ln)
        if m:
            blk = " ".join(ptx[i + 1:i + 4])
            st = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", blk)
            rg = re.search(r"Used (\d+) registers", blk)
            info[m.group(1)] = (rg.group(1) if rg else "?", st.groups() if st else ("?",) * 3)
    out = ["# SASS / ptxas summary of the step kernels (HEAD build)", "",
           "`cuobjdump -sass` of `paper_2511_02136_b200/libmlob.so` (sm_100a) and `nvcc -Xptxas -v` of "
           "`csrc/mlob_kernels.cu` (`python tools/sass_summary.py`).  Mnemonics that prove the hardware paths: "
           "`UBLKCP.S.G` = `cp.async.bulk` global->shared (TMA bulk copy), `UBLKCP.G.S` shared->global, "
           "`SYNCS.*` = mbarrier arrive / try-wait, `CREDUX` / `REDUX` = `redux.sync` warp reductions "
           "(uniform / vector destination), `VOTE` = ballots.", "",
           "| kernel | registers | stack / spill st / spill ld (B) | SASS instructions |", "|---|---|---|---|"]
    for f, name in KERNELS.items():
        r, (a, b, c) = info.get(f, ("?", ("?",) * 3))
        out.append(f"| {name} | {r} | {a} / {b} / {c} | {len(funcs.get(f, []))} |")
    out.append("")
    for f in list(KERNELS)[:2]:
        cnt = collections.Counter(x.split(".")[0] for x in funcs.get(f, []))
        full = collections.Counter(funcs.get(f, []))
        out += [f"## {KERNELS[f]}: opcode histogram (top 40)", "",
                " ".join(f"{k} {v};" for k, v in cnt.most_common(40)), "",
                "Key instructions: " + "; ".join(f"{k} x{full[k]}" for k in sorted(full) if k.startswith(KEY)), ""]
    path = os.path.join(ROOT, "profiles", "r2_sass_summary.md")
    open(path, "w").write("\n".join(out) + "\n")
    print(path)


if __name__ == "__main__":
    main()
