"""Helpers to load the committed golden fixtures (produced by oracle/gen_golden.py
from the unmodified reference)."""
import json
import math
from pathlib import Path

GOLDEN = Path(__file__).resolve().parent / "golden"


def fl(x):
    if x == "inf":
        return math.inf
    if x == "-inf":
        return -math.inf
    return float(x)


def load(name):
    return json.loads((GOLDEN / name).read_text())
