"""Markdown table of profiles/configs_r01.jsonl (tools/run_configs.sh output)
for DESIGN.md §5."""
import json
import sys

LABEL = {
    "c1-sw1-64": ("1: n=64", "SW¹"), "c2-sw1-4096": ("2: n=4096", "SW¹"),
    "c3-sw2-16384": ("3: n=16384", "SW² (⟨4,4,4;49⟩)"), "c3b-sw1-16384": ("3b: n=16384", "SW¹"),
    "c4a-ld1-13824": ("4a: n=13824", "Laderman¹"), "c4b-sw2-13824": ("4b: n=13824", "⟨4,4,4;49⟩"),
    "c5-sw2-32768": ("5: n=32768 (1-GPU leg)", "SW²"),
    "x-sw3-16384": ("n=16384, one more level", "SW³ (⟨8,8,8;343⟩)"),
    "x-ld2-13824": ("n=13824, one more level", "Laderman² (⟨9,9,9;529⟩)"),
    "x-sw3-32768": ("n=32768, one more level", "SW³"),
    "x-swld-13824": ("n=13824, mixed chain 2-then-3", "SW⊗LD (⟨6,6,6;161⟩)"),
    "x-ldsw-13824": ("n=13824, mixed chain 3-then-2", "LD⊗SW (⟨6,6,6;161⟩)"),
    "x-sw2-49152-bounded": ("n=49152, bounded workspace (85 GB cap)", "SW² (batches, generated K4/K6)"),
    "x-sw4-16384-hybrid": ("n=16384, four levels (hybrid)", "SW⁴: 1 level by level × 7 flattened SW³"),
    "x-sw4-32768-hybrid": ("n=32768, four levels (hybrid)", "SW⁴ (same)"),
    "x-sw5-32768-hybrid": ("n=32768, five levels (hybrid)", "SW⁵: 2 levels by level × 49 flattened SW³"),
}


def main(path="profiles/configs_r01.jsonl"):
    print("| Config | Triple / levels | TFLOPS | cuBLAS | Speedup | Leaf % of DMMA peak "
          "| Max scaled error | e2e stream / sync |")
    print("|---|---|---|---|---|---|---|---|")
    for line in open(path):
        d = json.loads(line)
        if d.get("failed"):
            continue
        c = d["config"]
        name, tri = LABEL.get(c["preset"], (c["preset"], c["triple"]))
        cl = d.get("classical", {})
        hyb = "hybrid" in c["preset"]
        e = d.get("e2e")
        e2e = f"{e['value']:.1f} / {e['sync']['value']:.1f}" if e and "sync" in e else "—"
        if c["preset"] == "c1-sw1-64":
            g = d.get("graph", {})
            print(f"| {name} | {tri} | launch-bound: {d['ms_per_step']:.3f} ms eager, "
                  f"**{g.get('ms_per_step', float('nan')):.4f} ms** as a CUDA graph (cuBLAS "
                  f"{cl.get('cublas_ms', float('nan')):.4f} ms) | — | — | — | "
                  f"{d['max_scaled_error']:.1e} | — |")
            continue
        print(f"| {name} | {tri} | {d['value']:.2f} | {cl.get('cublas_dgemm_tflops', float('nan')):.2f} "
              f"| {d.get('speedup_vs_cublas', float('nan')):.3f} | {100 * d['roofline']['frac']:.1f}"
              f"{'*' if hyb else ''} | {d['max_scaled_error']:.1e} | {e2e} |")


if __name__ == "__main__":
    main(*sys.argv[1:])
