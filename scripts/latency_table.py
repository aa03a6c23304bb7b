#!/usr/bin/env python3
"""Single-call evaluate() latency, reference vs drop-in (GPU box): runs
oracle/_ref/latency_on_reference and oracle/_ref/latency_on_b200 in each
GpuOptions mode and prints one JSON line per case with a "library" tag.

    python scripts/latency_table.py > profiles/r02_latency.jsonl
"""
import json
import os
import subprocess
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
RUNS = [("reference", "latency_on_reference", []),
        ("drop-in", "latency_on_b200", []),
        ("drop-in immutable_matrices", "latency_on_b200", ["immutable"]),
        ("drop-in resident", "latency_on_b200", ["resident"])]


def main():
    for tag, exe, args in RUNS:
        out = subprocess.run([os.path.join(ROOT, "oracle", "_ref", exe)] + args, capture_output=True, text=True,
                             timeout=600, check=True).stdout
        for line in out.splitlines():
            if line.startswith("{"):
                d = json.loads(line)
                d["library"] = tag
                print(json.dumps(d), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
