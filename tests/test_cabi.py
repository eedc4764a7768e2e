"""The C-ABI library loads on a CPU host and exports every symbol include/monet_b200.h declares.

No compute entry point is called here (no GPU); only the pure host functions
(version string, workspace-size queries, the arena planner) are exercised.
"""
import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

from paper_2010_14501_b200 import _native

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "monet_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(monet_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not _native.LIB_PATH.exists():
        from paper_2010_14501_b200 import build
        build.build()
    return _native.lib()


def test_header_symbols_exported(lib):
    syms = declared_symbols()
    assert len(syms) >= 30
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)], capture_output=True, text=True,
                         check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    # every declared symbol is also bound (with a signature) by the Python executor
    assert set(syms) <= set(_native.SIGNATURES), set(syms) - set(_native.SIGNATURES)


def test_exports_are_plain_c(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)], capture_output=True, text=True,
                         check=True).stdout
    # no C++-mangled monet symbols leak through the boundary
    assert not [l for l in out.splitlines() if "monet" in l and "_Z" in l.split()[-1]]


def test_host_queries(lib):
    assert lib.dll.monet_version().decode().endswith("sm_100a")
    d = _native.conv_desc(184, 56, 56, 64, 64, 3, 3, 1, 1)
    assert lib.dll.monet_conv_ws_bytes(0, 0, C.byref(d)) == 0           # implicit: no workspace
    ws = lib.dll.monet_conv_ws_bytes(1, 2, C.byref(d))                    # split-K wgrad partials
    assert ws > 0 and ws % (64 * 9 * 64 * 4) == 0
    assert lib.dll.monet_conv_ws_bytes(1, 3, C.byref(d)) >= ws            # bwd = max(dgrad, wgrad)
    bad = _native.conv_desc(1, 8, 8, 3, 8, 3, 3, 1, 1)                    # C % 4 != 0 is rejected
    assert lib.dll.monet_conv_ws_bytes(0, 0, C.byref(bad)) == 0
    assert lib.dll.monet_bn_scratch_bytes(1000, 64) > 0


def test_arena_plan_overlap_and_cap(lib):
    from paper_2010_14501_b200.engine import place_blocks
    blocks = [[1000, 0, 4], [500, 1, 3], [700, 2, 6], [1000, 4, 8]]
    peak, offs = place_blocks(blocks)
    for i, (si, ai, fi) in enumerate(blocks):
        for j, (sj, aj, fj) in enumerate(blocks):
            if i < j and ai < fj and aj < fi:     # live together -> disjoint
                assert offs[i] + si <= offs[j] or offs[j] + sj <= offs[i]
    assert peak >= 1008 + 512 + 704  # blocks 0-2 live together, each rounded to 16 B (ARENA_ALIGN)
    assert all(o % 16 == 0 for o in offs)
    from paper_2010_14501_b200.engine import BudgetExceeded
    with pytest.raises(BudgetExceeded):
        place_blocks(blocks, capacity=1000)


def test_public_abi_has_no_debug_hooks(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)], capture_output=True, text=True,
                         check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    assert not [s for s in exported if s.startswith("monet_debug")]
    assert "monet_profile_variant" in exported


def test_prof_desc_layout_matches_header():
    # monet_prof_desc: op, pass, conv (13 ints), conv_needs_dx, then int64 rows (8-aligned), c
    assert C.sizeof(_native.ConvDesc) == 13 * 4
    assert _native.ProfDesc.rows.offset == 8 + 13 * 4 + 4
    assert C.sizeof(_native.ProfDesc) == 80
