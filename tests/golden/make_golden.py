"""Generates the golden fixtures in tests/golden from the UNMODIFIED reference
library (oracle/_ref/libgravitree_ref.so, built in place from /root/reference
by oracle/Makefile).  Run from the repo root:  python tests/golden/make_golden.py

Each fixture holds the reference's own outputs for one input:
  mass/pos/vel      sample_model(name, n, seed=1)            models.cpp:442-460
  tree_*            build_tree(leaf_cap 8)                    octree.cpp:51-162
  boot_acc, acc_old_mag  GravityEngine::bootstrap (direct)    engine.cpp:89-103
  acc, events       build + evaluate(all), eps 2^-5, dacc 2^-9 engine.cpp:31-81
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.refpy import Ref  # noqa: E402


def make(name, model, n):
    r = Ref()
    mass, pos, vel = r.sample_model(model, n, 1)
    t = r.build_tree(mass, pos)
    e = r.engine(eps=2.0 ** -5, dacc=2.0 ** -9, threads=4)
    boot_acc, amag, _ = e.bootstrap(mass, pos)
    e.build(mass, pos)
    acc, _, ev = e.evaluate(mass, pos, amag)
    out = dict(mass=mass, pos=pos, vel=vel, boot_acc=boot_acc, acc_old_mag=amag, acc=acc,
               events=np.array([ev["interactions"], ev["mac_evals"], ev["list_pushes"]], np.uint64))
    for k in ("bbox", "keys", "perm", "rank", "cells", "depth", "nodes"):
        out["tree_" + k] = getattr(t, k)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(name, {k: v.shape for k, v in out.items()}, ev)


if __name__ == "__main__":
    make("plummer_4096", "plummer", 4096)
    make("m31_16384", "m31", 16384)
