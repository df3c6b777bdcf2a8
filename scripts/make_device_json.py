"""Write tests/golden/device_guadalupe_like.json: a synthetic 16-qubit heavy-hex calibration
snapshot (workloads.synthetic_device; the ranges of DESIGN.md §3's input recipe) in the SPEC
S:365-370 schema.  Synthetic numbers, not a real device."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402

if __name__ == "__main__":
    out = os.path.join(ROOT, "tests", "golden", "device_guadalupe_like.json")
    with open(out, "w") as f:
        json.dump(W.synthetic_device(), f, indent=1)
    print(out)
