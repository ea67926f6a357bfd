"""SASS + PTX instruction-diversity report over the compiled variants.

Reproduces the paper's code analysis (ref/PAPER.md:133-140: unique mnemonics and total
instruction count per compiled configuration, best config marked) for the sm_100a attention
variants, using the UNMODIFIED reference statistics (`ktune analyze-asm`,
ref/pkg/src/ktune/asmstats.py:73-207, ref/pkg/src/ktune/cli.py:444-470).

    python scripts/asm_diversity.py [--best prefill_BM256_BN128_S3] [--tag r01]

Inputs: ``cuobjdump -sass`` of libb200attn.so split per kernel (instruction lines only) and
``nvcc -ptx`` of csrc/capi.cu split per ``.entry``.  Each document is named after the space
point it implements (prefill: BLOCK_M/BLOCK_N/num_stages; decode: TILE_N/num_stages/GQA).
Outputs: profiles/<tag>_asm_diversity_{sass,ptx}.{csv,json} + a markdown table.
"""

from __future__ import annotations

import argparse
import json
import os
import re
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
REF = ROOT / "baseline" / "_ref"
LIB = ROOT / "paper_2505_03780_b200" / "_lib" / "libb200attn.so"
CAPI = ROOT / "paper_2505_03780_b200" / "csrc" / "capi.cu"

_TEMPLATE = re.compile(r"b200(\d+)([a-z_]+)ILi(\d+)ELi(\d+)E(?:Li(\d+)E)?(?:Li(\d+)E)?")


def variant_id(mangled: str) -> str | None:
    """prefill_fwd_kernel<NQ,BN,NS,EMU,SPLIT> -> prefill_BM{128*NQ}_BN{BN}_S{NS}_W{4*SPLIT};
    decode_flat_kernel<G,NS,FP8> -> decode_T16_G{G}_S{NS}[_fp8]; decode_split_kernel<NS> -> decode_T128_S{NS}."""
    m = re.search(r"prefill_fwd_kernelILi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)E", mangled)
    if m:
        return f"prefill_BM{128 * int(m.group(1))}_BN{m.group(2)}_S{m.group(3)}_W{4 * int(m.group(5))}"
    m = re.search(r"decode_flat_kernelILi(\d+)ELi(\d+)ELb(\d)E", mangled)
    if m:
        return f"decode_T16_G{m.group(1)}_S{m.group(2)}" + ("_fp8" if m.group(3) == "1" else "")
    m = re.search(r"decode_split_kernelILi(\d+)E", mangled)
    if m:
        return f"decode_T128_S{m.group(1)}"
    return None


def split_sass(text: str) -> dict[str, str]:
    docs, cur, buf = {}, None, []
    for line in text.splitlines():
        if "Function :" in line:
            if cur:
                docs[cur] = "\n".join(buf)
            cur, buf = variant_id(line.split("Function :")[1].strip()), []
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(.*?)\s*;", line)
        if m:
            buf.append(m.group(1) + " ;")
    if cur:
        docs[cur] = "\n".join(buf)
    return {k: v for k, v in docs.items() if k}


def split_ptx(text: str) -> dict[str, str]:
    docs = {}
    parts = re.split(r"\n(?=\.visible \.entry |\.entry |\.weak \.entry )", text)
    for p in parts:
        m = re.match(r"\.(?:visible |weak )?\.?entry (\S+)\(", p) or re.match(r"\.(?:visible |weak )\.entry (\S+)\(", p)
        if not m:
            continue
        vid = variant_id(m.group(1))
        if vid:
            # keep only the body (directives/params are skipped by the analyser anyway)
            docs[vid] = p[p.find("{"):] if "{" in p else p
    return docs


def run_ktune(docs: dict[str, str], kind: str, suffix: str, best: str | None, prefix: Path) -> dict:
    with tempfile.TemporaryDirectory() as d:
        for k, v in docs.items():
            (Path(d) / f"{k}{suffix}").write_text(v)
        env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(REF), str(ROOT)]))
        args = [sys.executable, "-m", "ktune", "analyze-asm", d, "-o", str(prefix), "--no-plot"]
        if best and best in docs:
            args += ["--best", best]
        r = subprocess.run(args, env=env, capture_output=True, text=True)
        if r.returncode != 0:
            raise SystemExit(f"ktune analyze-asm ({kind}) failed: {r.stdout}{r.stderr}")
        print(r.stdout.strip())
    return json.loads(Path(str(prefix) + ".json").read_text())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--best", default="prefill_BM256_BN128_S3", help="variant the tuner picked for the marker")
    ap.add_argument("--tag", default="r01")
    a = ap.parse_args()
    sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True, check=True).stdout
    from paper_2505_03780_b200 import build

    with tempfile.TemporaryDirectory() as d:
        ptx_path = Path(d) / "capi.ptx"
        flags = [f for f in build.FLAGS if f not in ("-shared", "-Xcompiler", "-fPIC", "-lineinfo")]
        flags = [f.replace("code=sm_100a", "code=compute_100a") for f in flags]
        subprocess.run([build.NVCC, *flags, "-ptx", "-o", str(ptx_path), str(CAPI)], check=True)
        ptx = ptx_path.read_text()
    out = {}
    sass_docs = split_sass(sass)
    for kind, docs, suffix in (("sass", sass_docs, ".asm"), ("ptx", split_ptx(ptx), ".ptx")):
        prefix = ROOT / "profiles" / f"{a.tag}_asm_diversity_{kind}"
        out[kind] = run_ktune(docs, kind, suffix, a.best, prefix)
    md = ["# Instruction diversity of the compiled sm_100a variants (ktune analyze-asm, unmodified)", "",
          "Per variant: unique mnemonics (opcode + all suffixes) and total static instructions, for the SASS",
          "that runs and the PTX it was lowered from (ref/PAPER.md:133-140 ran the same analysis on PTX).", "",
          "| variant | SASS unique | SASS total | PTX unique | PTX total |", "|---|---|---|---|---|"]
    sass_rows = {r["id"]: r for r in out["sass"]["sources"]}
    ptx_rows = {r["id"]: r for r in out["ptx"]["sources"]}
    for vid in sorted(set(sass_rows) | set(ptx_rows)):
        s, p = sass_rows.get(vid, {}), ptx_rows.get(vid, {})
        mark = " (best C3)" if vid == a.best else ""
        md.append(f"| {vid}{mark} | {s.get('unique')} | {s.get('total')} | {p.get('unique')} | {p.get('total')} |")
    for vid in (a.best, "decode_T16_G4_S5"):
        body = sass_docs.get(vid, "")
        ops = [t for ln in body.splitlines() for t in ln.split()[:2] if not t.startswith("@")][::1]
        tc = sorted({t for t in ops if t.startswith(("UTC", "UTMA", "UBLKCP", "SYNCS", "LDTM", "STTM"))})
        md += ["", f"{vid}: tcgen05 / TMA / mbarrier SASS mnemonics: {', '.join(tc)}"]
    (ROOT / "profiles" / f"{a.tag}_asm_diversity.md").write_text("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
