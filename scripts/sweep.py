"""Configuration sweep for the BASELINE.json configs (run under gpurun):
hybrid vs same-GPU full attention, algorithmic GB/s, per workload / retrieval
fraction / top-k.  Prints one markdown table row per case (and JSON lines to
gpurun_out/sweep.jsonl)."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CASES = [
    # (workload, retrieval fraction, top-k override)
    ("llama3-8b-32k", 0.125, None),
    ("llama3-8b-128k", 0.125, None),
    ("qwen3-8b-128k", 0.125, None),
    ("qwen3-8b-128k", 0.25, None),
    ("qwen3-8b-128k", 0.5, None),
    ("llama3-8b-64k-b16", 0.125, 512),
    ("llama3-8b-64k-b16", 0.125, 2048),
    ("llama3-8b-64k-b16", 0.125, 8192),
]


def main():
    out = open(ROOT / "gpurun_out" / "sweep.jsonl", "w")
    print("| workload | retrieval frac | top-k | hybrid us/token | full us/token | speedup | "
          "algorithmic GB/s | frac of peak |")
    print("|---|---|---|---|---|---|---|---|")
    for wl, frac, k in CASES:
        cmd = [sys.executable, str(ROOT / "bench.py"), "--workload", wl, "--steps", "10",
               "--warmup", "3", "--no-cpu-baseline", "--retrieval-frac", str(frac)]
        if k:
            cmd += ["--top-k", str(k)]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        try:
            d = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception:
            print(f"| {wl} | {frac} | {k} | FAILED: {r.stderr[-200:]!r} |")
            continue
        out.write(json.dumps(d) + "\n")
        f = d["full_attention"]
        print(f"| {wl} | {frac} | {d['config']['top_k']} | {d['value']:.1f} | "
              f"{f['us_per_token']:.1f} | {f['speedup_hybrid_vs_full']:.2f}x | "
              f"{d['roofline']['achieved']:.0f} | {d['roofline']['frac']:.3f} |", flush=True)


if __name__ == "__main__":
    main()
