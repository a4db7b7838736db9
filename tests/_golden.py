"""Loader for tests/golden/golden.json (made from the compiled reference by
tests/golden/make_golden.py)."""
import hashlib
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden", "golden.json")


def load():
    with open(GOLDEN) as f:
        return json.load(f)


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def points(recipe) -> np.ndarray:
    k = recipe["kind"]
    if k == "arange":
        return np.arange(recipe["n"], dtype=np.float32).reshape(-1, 1)
    if k == "explicit":
        return np.asarray(recipe["values"], np.float32)
    if k == "random":
        rng = np.random.default_rng(recipe["seed"])
        return rng.random((recipe["n"], recipe["d"]), dtype=np.float32) * np.float32(recipe["scale"])
    if k == "synthetic":
        from paper_2006_06743_b200 import synthetic
        return synthetic.generate(recipe["cfg"], n=recipe["n"])
    raise KeyError(k)


def cases():
    return load()["cases"]
