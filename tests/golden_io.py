"""Loads tests/golden/reference_vectors.npz (made by tests/golden/make_golden.py
from the unmodified reference) as {section: {name: array}}."""
import os

import numpy as np

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_vectors.npz")


def load():
    z = np.load(PATH)
    out = {}
    for key in z.files:
        sec, name = key.split("__", 1)
        out.setdefault(sec, {})[name] = z[key]
    return out
