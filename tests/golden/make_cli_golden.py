"""Outputs of the REAL reference CLI (normint/cli.py) on the committed file
fixtures, for the GPU CLI parity test (tests/test_gpu_cli.py).  Run in the
build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_cli_golden.py

Each case writes <name>.depth.pfm and <name>.jsonl (the diagnostics records,
wall_ms dropped) under tests/golden/cli/; ``decompose`` writes the label blob.
"""

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
FILES = os.path.join(HERE, "files")
OUT = os.path.join(HERE, "cli")

from normint import cli  # noqa: E402

# name: extra integrate flags (inputs: files/normals.{pfm,png}, mask, intrinsics)
CASES = {
    "default_pfm": ["--normals", "normals.pfm"],
    "png_mask_merge2": ["--normals", "normals.png", "--mask", "mask.png", "--merge-freq", "2"],
    "hard_gauge": ["--normals", "normals.pfm", "--reweighting", "hard", "--gauge-depth", "2.5"],
    "bini4_off": ["--normals", "normals.pfm", "--connectivity", "4", "--continuity-model", "bini",
                  "--reweighting", "off", "--theta-c", "5"],
    "pixel_baseline": ["--normals", "normals.png", "--pixel-baseline", "--max-iters", "30"],
    "theta_none": ["--normals", "normals.pfm", "--theta-c", "none", "--max-iters", "20"],
}


def _args(name, flags):
    fl = []
    for f in flags:
        fl.append(os.path.join(FILES, f) if f.endswith((".pfm", ".png")) else f)
    return ["integrate", *fl, "--intrinsics", os.path.join(FILES, "intrinsics.json"),
            "--output", os.path.join(OUT, f"{name}.depth.pfm"),
            "--diagnostics", os.path.join(OUT, f"{name}.jsonl")]


def main():
    os.makedirs(OUT, exist_ok=True)
    for name, flags in CASES.items():
        rc = cli.main(_args(name, flags))
        assert rc == 0, (name, rc)
        path = os.path.join(OUT, f"{name}.jsonl")
        recs = [json.loads(x) for x in open(path)]
        for r in recs:
            r.pop("wall_ms", None)
        with open(path, "w") as fh:
            fh.writelines(json.dumps(r) + "\n" for r in recs)
    rc = cli.main(["decompose", "--normals", os.path.join(FILES, "normals.png"), "--mask",
                   os.path.join(FILES, "mask.png"), "--output", os.path.join(OUT, "decomp")])
    assert rc == 0
    os.remove(os.path.join(OUT, "decomp.labels.png"))  # the PNG is a hash of the blob
    json.dump(CASES, open(os.path.join(OUT, "cases.json"), "w"), indent=1)
    print("written", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    sys.exit(main())
