"""Reader for the fixtures written by tests/golden/make_golden.py."""

import os

import numpy as np

DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


class Fixture:
    def __init__(self, name):
        self.z = dict(np.load(os.path.join(DIR, name)))

    def count(self, key):
        return self.z[key + "__off"].size - 1

    def get(self, key, i):
        off = self.z[key + "__off"]
        return self.z[key][off[i]:off[i + 1]]

    def vec(self, key, i):
        return self.get(key, i).reshape(-1)

    def scalar(self, key, i):
        return float(self.get(key, i).reshape(-1)[0])

    def graph_arrays(self, i):
        e = self.get("edges", i).astype(np.int64).reshape(-1, 2)
        return int(self.scalar("n", i)), e[:, 0].copy(), e[:, 1].copy(), self.vec("costs", i).astype(np.float64)


def load(name):
    return Fixture(name)
