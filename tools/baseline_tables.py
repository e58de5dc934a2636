"""Render BASELINE.md's per-config table from a tools/run_configs.py JSONL file.

    python tools/baseline_tables.py profiles/r2_configs.jsonl
"""
import json
import sys


def fmt_ms(x):
    if x is None:
        return "—"
    return f"{x:,.0f}" if x >= 100 else (f"{x:.1f}" if x >= 10 else f"{x:.2f}")


def main(path):
    import os

    rows = [json.loads(l) for l in open(path) if l.strip().startswith("{")]
    mp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "c5", "manifest.json")
    man = json.load(open(mp)) if os.path.exists(mp) else {}
    print("| Config | step ms (build + pairs) | pair-intersections/s | frequent pairs | K2 ms | K2 % R_int "
          "| K1 insertions/s | parity | CPU horizontal oracle s | dense XᵀX ms | GPU merge ms |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    def cpu_s(r):
        if "golden" in r.get("parity", "") and r["config"] in man:
            e = man[r["config"]]
            return f"{e['horizontal_s']} ({e['threads']} thr, golden)"
        return r.get("oracle_s", "—")

    for r in rows:
        d = r.get("dense_xtx")
        m = r.get("merge")
        k1 = r.get("k1") or {}
        ins = k1.get("insertions_per_s")
        par = "bit-exact" if r["exact"] else "**MISMATCH**"
        how = r.get("parity", "")
        if "golden" in how:
            par += " (full-size golden)"
        elif "horizontal" in how:
            par += " (horizontal oracle)"
        else:
            par += f" ({how})"
        print(f"| {r['config']} n={r['n']:,} m={r['m']:,} s={r['threshold']} "
              f"| {fmt_ms(r['step_ms'])} ({fmt_ms(r['build_ms'])} + {fmt_ms(r['pairs_ms'])}) "
              f"| {r['pairs_per_s']:.2e} | {r['K']:,} | {fmt_ms(r['k2_ms'])} | {100 * (r['k2_frac_R_int'] or 0):.0f} % "
              f"| {ins:.1e} | {par} | {cpu_s(r)} "
              f"| {fmt_ms(d['total_ms']) if d else 'n/a'} | {fmt_ms(m['kernel_ms']) if m else '—'} |")
    pf = [r for r in rows if r.get("prefiltered")]
    for r in pf:
        p = r["prefiltered"]
        print(f"\n{r['config']} with the P:118 pre-filter: {p['frequent_items']:,} frequent items, "
              f"{fmt_ms(p['total_ms'])} ms (filter + select + build {fmt_ms(p['build_ms'])} + pairs "
              f"{fmt_ms(p['pairs_ms'])}), equal to the unfiltered output: {p['equal_to_unfiltered']}")


if __name__ == "__main__":
    main(sys.argv[1])
