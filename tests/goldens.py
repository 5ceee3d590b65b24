"""Loading helpers for the committed golden vectors (tests/golden/)."""

import gzip
import json
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    path = os.path.join(GOLDEN, name)
    if name.endswith(".gz"):
        with gzip.open(path, "rt") as f:
            return json.load(f)
    with open(path) as f:
        return json.load(f)


def replay(name, mode):
    path = f"replay_{name}_{mode}.json.gz"
    if not os.path.exists(os.path.join(GOLDEN, path)):
        return None
    return load(path)


def digests():
    return load("replay_digests.json")
