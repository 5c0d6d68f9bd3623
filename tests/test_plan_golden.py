"""Planner/simulator parity: the SAME driver source (tests/cpp/plan_dump.cpp,
written only against the reference `shardplan` headers) compiled against this
repo's drop-in library must print byte-identical output to the compiled
reference (tests/golden/plan_dump.txt.gz, made by make_plan_golden.sh).
Doubles print as %a, so identical means bit-exact — SURVEY.md §8(a) rows
a1-a16 and §8(c) row c2."""
import gzip
import os
import subprocess
from pathlib import Path

import pytest

from paper_2311_00257_b200 import build

REPO = Path(__file__).resolve().parents[1]
GOLDEN = REPO / "tests" / "golden" / "plan_dump.txt.gz"


@pytest.fixture(scope="module")
def dump_binary(tmp_path_factory):
    lib = build.build_library()
    out = tmp_path_factory.mktemp("dump") / "plan_dump"
    cmd = [build.CXX, "-std=c++20", "-O1", "-I", str(REPO / "include"),
           str(REPO / "tests" / "cpp" / "plan_dump.cpp"), "-o", str(out),
           "-L", str(lib.parent), "-lamsp", f"-Wl,-rpath,{lib.parent}"]
    subprocess.run(cmd, check=True, capture_output=True)
    return out


def _section(binary, name):
    r = subprocess.run([str(binary), name], capture_output=True, text=True, check=True)
    return r.stdout


def _golden_sections():
    text = gzip.decompress(GOLDEN.read_bytes()).decode()
    parts, cur, name = {}, [], None
    for line in text.splitlines(keepends=True):
        if line.startswith("## "):
            if name:
                parts[name] = "".join(cur)
            name, cur = line[3:].strip(), [line]
        else:
            cur.append(line)
    parts[name] = "".join(cur)
    return parts


GOLD = _golden_sections()


@pytest.mark.parametrize("section", ["comm", "domain", "cost", "planner", "sim", "placement"])
def test_section_bit_exact(dump_binary, section):
    mine = _section(dump_binary, section)
    ref = GOLD[section]
    if mine != ref:
        a, b = mine.splitlines(), ref.splitlines()
        for i, (x, y) in enumerate(zip(a, b)):
            if x != y:
                pytest.fail(f"{section}: first difference at line {i}:\n mine: {x[:400]}\n  ref: {y[:400]}")
        pytest.fail(f"{section}: length differs ({len(a)} vs {len(b)} lines)")


def test_golden_covers_every_entry_point():
    """The fixture exercises every public reference function (a1-a16 + placement)."""
    text = "".join(GOLD.values())
    for key in ["\nring ", "eff ar", "fallback", "csv ", "json ", "synthetic", "validate cluster",
                "preset ", "cost ", "greedy ", "flops ", "enum ", "solve ", "oracle ",
                "compare ", "sim ", "simL ", "simulate ", "trace one", "assign ", "cross "]:
        assert key in text, key
