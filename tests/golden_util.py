"""Helpers to read the golden fixtures (binary64 little-endian hex, runlog.py:21-27)."""
import json
import struct
from functools import lru_cache
from pathlib import Path

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=None)
def load(name: str):
    with open(GOLDEN / name, encoding="utf-8") as fh:
        return json.load(fh)


def hf(h: str) -> float:
    return struct.unpack("<d", bytes.fromhex(h))[0]


def hfl(hs) -> list:
    return [hf(h) for h in hs]


def fh(v: float) -> str:
    return struct.pack("<d", v).hex()


def fhl(vs) -> list:
    return [fh(float(v)) for v in vs]


def u64(h: str) -> int:
    return int(h, 16)
