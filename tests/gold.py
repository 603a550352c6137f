"""Golden-fixture loading shared by the CPU and GPU parity tests."""
import json
import os

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
STATUS_NAMES = ("inserted", "duplicate_key", "table_full", "invalid_key", "out_of_memory")

_cache = {}


def load(name):
    if name not in _cache:
        with open(os.path.join(GOLD, name)) as fh:
            _cache[name] = json.load(fh)
    return _cache[name]


def ints(xs):
    return [int(x) for x in xs]
