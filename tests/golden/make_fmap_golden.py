"""Generate tests/golden/fmap/: FMAP files written by the REAL reference (its own CLI).

Run here (not on the GPU box -- /root/reference and baseline/_ref do not travel there):

    python tests/golden/make_fmap_golden.py

Uses the unmodified reference package installed in baseline/_ref (DESIGN.md recipe) with its
compiled backend, driven through its CLI (`python -m denseprop.cli`, cli.py:150-206):

  fixture --kind random-small   -> random-small.net, conv1/conv2 .weights.fmap, image.fmap
                                   (fixtures.py:106-134, weight files netspec.py:123-150)
  forward --dtype 32            -> forward.fmap (the dense output, cli.py:180-191)
  backward --dtype 32 --input-grad with a 40-pixel mask file
                                -> grads/layerKK.kernel.fmap (multi-record), .bias.fmap,
                                   input_delta.fmap (cli.py:194-221)
plus the same two runs on a relu variant of the spec (random-small-relu.net ->
forward_relu.fmap, grads_relu/), target.fmap written with the reference's fmap.write_fmap from a float64 map (the
float64 -> float32 conversion on write) and mask.txt.  Sizes are kept small (a few KB).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
OUT = os.path.join(HERE, "fmap")
REF = os.path.join(REPO, "baseline", "_ref")


def cli(*args):
    env = dict(os.environ, PYTHONPATH=REF, DENSEPROP_BACKEND="compiled")
    subprocess.run([sys.executable, "-m", "denseprop.cli", *args], check=True, env=env,
                   cwd=OUT, stdout=subprocess.DEVNULL)


def main():
    if os.path.isdir(OUT):
        shutil.rmtree(OUT)
    os.makedirs(OUT)
    cli("fixture", "--kind", "random-small", "--seed", "3", "--out", ".")
    cli("forward", "--spec", "random-small.net", "--image", "image.fmap", "--out",
        "forward.fmap", "--dtype", "32", "--backend", "compiled")
    sys.path.insert(0, REF)
    from denseprop import fmap as ref_fmap
    out = ref_fmap.read_fmap(os.path.join(OUT, "forward.fmap"))
    rng = np.random.default_rng(5)
    ref_fmap.write_fmap(os.path.join(OUT, "target.fmap"),
                        rng.uniform(-1, 1, out.shape).astype(np.float64))
    h, w = out.shape[1:]
    pix = rng.choice(h * w, 40, replace=False)
    with open(os.path.join(OUT, "mask.txt"), "w") as fh:
        fh.write("".join(f"{int(p) // w} {int(p) % w}\n" for p in sorted(pix)))
    cli("backward", "--spec", "random-small.net", "--image", "image.fmap", "--target",
        "target.fmap", "--mask", "mask.txt", "--out", "grads", "--input-grad", "--dtype", "32",
        "--backend", "compiled")
    # relu variant of the same fixture: every op bit-reproducible (no numpy tanh), so this
    # repo's exact tier must write byte-identical forward / gradient files
    with open(os.path.join(OUT, "random-small.net")) as fh:
        text = fh.read().replace("nonlin kind=tanh", "nonlin kind=relu")
    with open(os.path.join(OUT, "random-small-relu.net"), "w") as fh:
        fh.write(text)
    cli("forward", "--spec", "random-small-relu.net", "--image", "image.fmap", "--out",
        "forward_relu.fmap", "--dtype", "32", "--backend", "compiled")
    cli("backward", "--spec", "random-small-relu.net", "--image", "image.fmap", "--target",
        "target.fmap", "--mask", "mask.txt", "--out", "grads_relu", "--input-grad", "--dtype",
        "32", "--backend", "compiled")
    for root, _, files in os.walk(OUT):
        for f in sorted(files):
            p = os.path.join(root, f)
            print(os.path.relpath(p, OUT), os.path.getsize(p))


if __name__ == "__main__":
    main()
