"""Builds kernel variants (macro settings) as separate .so files for A/B timing."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_05370_b200 import build as B  # noqa: E402

VARIANTS = {
    "fm3": ["-DHSIM_FINAL_MULT=3"],
    "prio4": ["-DHSIM_PRIO4"],
    "norq2": ["-DHSIM_REQ_MINJOBS=(1LL<<40)"],
    "fp3": ["-DHSIM_FINALP_MINB=3"],
    "mp8": ["-DHSIM_MULTI_PMAX=8"],
    "mp9": ["-DHSIM_MULTI_PMIN=9"],
    "mlp": ["-DHSIM_MULTI_STREAM=3"],
    "mg2": ["-DHSIM_MULTI_GRIDDIV=2"],
    "mg4": ["-DHSIM_MULTI_GRIDDIV=4"],
    "mm20": ["-DHSIM_MULTI_MAXJOBS=(1LL<<20)"],
    "mm0": ["-DHSIM_MULTI_MAXJOBS=0"],
    "mm22": ["-DHSIM_MULTI_MAXJOBS=(1LL<<22)"],
    "sp6": ["-DHSIM_SPLIT_MINB=6"],
    "sp8": ["-DHSIM_SPLIT_MINB=8"],
    "sp4": ["-DHSIM_SPLIT_MINB=4"],
    "sp5": ["-DHSIM_SPLIT_MINB=5"],
    "rq5": ["-DHSIM_REQ_MINP=5"],
    "rq4": ["-DHSIM_REQ_MINP=4"],
    "rq4d8": ["-DHSIM_REQ_MINP=4", "-DHSIM_DEFER_MIN=8"],
    "rq4d32": ["-DHSIM_REQ_MINP=4", "-DHSIM_DEFER_MIN=32"],
    "rq2": ["-DHSIM_REQ_MINP=2"],
    "fm16": ["-DHSIM_FINAL_MULT=16"],
    "fm12": ["-DHSIM_FINAL_MULT=12"],
    "fm6": ["-DHSIM_FINAL_MULT=6"],
    "nb2": ["-DHSIM_NBATCH=2"],
    "nb3": ["-DHSIM_NBATCH=3"],
    "nb4": ["-DHSIM_NBATCH=4"],
    "rq1": ["-DHSIM_DEFER_MIN=1", "-DHSIM_REQ_MINP=2", "-DHSIM_REQ_MINJOBS=0"],
    "norq": ["-DHSIM_REQ_MAXP=1"],
    "rq64": ["-DHSIM_DEFER_MIN=64"],
    "rqmin2": ["-DHSIM_REQ_MINP=2"],
    "rqmin4": ["-DHSIM_REQ_MINP=4"],
    "s4": ["-DHSIM_SYNC_MINB=4"],
    "s5": ["-DHSIM_SYNC_MINB=5"],
    "s3": ["-DHSIM_SYNC_MINB=3"],
    "w16": ["-DHSIM_WHOLE_MAXP=16"],
    "pm6": ["-DHSIM_PIPE_MINB=6"],
    "pm7": ["-DHSIM_PIPE_MINB=7"],
    "nb1": ["-DHSIM_NBATCH=1"],
    "s7": ["-DHSIM_SYNC_MINB=7"],
    "noprio": ["-DHSIM_NOPRIO"],
    "deepfirst": ["-DHSIM_DEEPFIRST"],
    "w8": ["-DHSIM_WHOLE_MAXP=8"],
    "fm4": ["-DHSIM_FINAL_MULT=4"],
    "fm2": ["-DHSIM_FINAL_MULT=2"],
    "aff11": ["-DHSIM_AFFINE_MAXP=11"],
    "aff16": ["-DHSIM_AFFINE_MAXP=16"],
    "pm5": ["-DHSIM_PIPE_MINB=5"],
    "pm4": ["-DHSIM_PIPE_MINB=4"],
    "noaff": ["-DHSIM_AFFINE_MAXP=0"],
    "aff4": ["-DHSIM_AFFINE_MAXP=4", "-DHSIM_PIPE_MINB=6"],
    "aff12": ["-DHSIM_AFFINE_MAXP=12", "-DHSIM_PIPE_MINB=6"],
    "u4": ["-DHSIM_UNROLL_MAXP=4"],
    "u6": ["-DHSIM_UNROLL_MAXP=6"],
    "u16": ["-DHSIM_UNROLL_MAXP=16"],
    "p8s6": ["-DHSIM_PIPE_MINB=8", "-DHSIM_SYNC_MINB=6"],
    "wcells": ["-DHSIM_WARPCELLS"],
    "diag": ["-DHSIM_DIAG"],
    "noskip": ["-DHSIM_NOSKIP"],
    "noskip_wc": ["-DHSIM_NOSKIP", "-DHSIM_WARPCELLS"],
    "nb6": ["-DHSIM_NBATCH=6"],
    "nb8": ["-DHSIM_NBATCH=8"],
    "p6s5": ["-DHSIM_PIPE_MINB=6", "-DHSIM_SYNC_MINB=5"],
    "p7s4": ["-DHSIM_PIPE_MINB=7", "-DHSIM_SYNC_MINB=4"],
    "fp6": ["-DHSIM_FINALP_MINB=6"],
    "fp4": ["-DHSIM_FINALP_MINB=4"],
    "fp1": ["-DHSIM_FINALP_MINB=1"],
    "f8_nb": ["-DHSIM_FASTP=8"],
    "f8_b3": ["-DHSIM_FASTP=8", "-DHSIM_MINB=3"],
    "f4_b4": ["-DHSIM_FASTP=4", "-DHSIM_MINB=4"],
    "f8_b4": ["-DHSIM_FASTP=8", "-DHSIM_MINB=4"],
    "f4_b6": ["-DHSIM_FASTP=4", "-DHSIM_MINB=6"],
    "f4_b8": ["-DHSIM_FASTP=4", "-DHSIM_MINB=8"],
    "f2_b8": ["-DHSIM_FASTP=2", "-DHSIM_MINB=8"],
}
out_dir = os.path.join(B.PKG, "variants")
os.makedirs(out_dir, exist_ok=True)
names = sys.argv[1:] or list(VARIANTS)
for name in names:
    out = os.path.join(out_dir, f"libhsim_{name}.so")
    cmd = B.nvcc_cmd(out=out, extra=tuple(VARIANTS[name]) + ("-Xptxas", "-v"))
    r = subprocess.run(cmd, capture_output=True, text=True)
    lines = r.stderr.splitlines()
    info = [lines[k + 1].strip() + " | " + lines[k + 2].strip() for k, l in enumerate(lines)
            if "Function properties for _ZN4hsim6k_eval" in l and k + 2 < len(lines)]
    print(name, r.returncode, info)
