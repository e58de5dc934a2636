"""Host-side checks of the C-ABI library (no GPU needed): it loads, exports every symbol
include/batmap.h declares, rejects bad arguments without touching the device, and its
host-only planner partitions the pair triangle exactly."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    hdr = open(os.path.join(ROOT, "include", "batmap.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:batmap_status|void|const char\*)\s+(batmap_\w+)\s*\(", hdr, flags=re.M)))


def test_library_exports_every_declared_symbol():
    from paper_1102_1003_b200 import batmap

    lib = batmap.load_library()
    names = _declared_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    raw = ctypes.CDLL(batmap.LIB_PATH)
    for n in names:
        getattr(raw, n)
    assert batmap.version().startswith("batmap-b200")


def test_library_is_sm100a_only():
    from paper_1102_1003_b200 import batmap
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", batmap.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    dump = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", batmap.LIB_PATH],
                          capture_output=True, text=True).stdout
    funcs = dump.split("Function : ")
    k2 = [f for f in funcs if f.startswith("_ZN2bm8k2_tiled")]
    assert k2, "tiled intersection kernel missing"
    sass = "".join(k2)
    assert "UTMALDG" in sass  # TMA (cp.async.bulk.tensor) in the intersection kernel
    assert "IDP.4A" in sass and "LOP3" in sass


def test_argument_errors_without_device():
    from paper_1102_1003_b200 import batmap

    lib = batmap.load_library()
    h = ctypes.c_void_p()
    assert lib.batmap_build(None, None, 3, 10, None, None, ctypes.byref(h)) == batmap.BATMAP_E_INVALID
    assert b"NULL" in lib.batmap_last_error()
    assert lib.batmap_build(ctypes.c_void_p(8), ctypes.c_void_p(8), 3, 1 << 31, None, None,
                            ctypes.byref(h)) == batmap.BATMAP_E_OVERFLOW
    o = batmap.BuildOpts()
    o.r_min = 96
    assert lib.batmap_build(ctypes.c_void_p(8), ctypes.c_void_p(8), 3, 10, ctypes.byref(o), None,
                            ctypes.byref(h)) == batmap.BATMAP_E_INVALID
    n = ctypes.c_int64()
    assert lib.batmap_pair_supports(None, None, 0, 1, None, 0, ctypes.byref(n), None) == batmap.BATMAP_E_INVALID
    inf = batmap.Info()
    assert lib.batmap_info(None, ctypes.byref(inf)) == batmap.BATMAP_E_INVALID
    lib.batmap_destroy(None)


def _all_tiles(class_n, tile_m):
    out = set()
    C = len(class_n)
    for a in range(C):
        for b in range(a, C):
            ta, tb = -(-class_n[a] // tile_m), -(-class_n[b] // tile_m)
            for i in range(ta):
                for j in range(i if a == b else 0, tb):
                    out.add((a, b, i, j))
    return out


@pytest.mark.parametrize("class_n,class_w", [([1000], [192]), ([7800, 2200], [1536, 3072]),
                                             ([99835, 40, 30, 20, 10, 5, 3, 1], [6144 * 2 ** k for k in range(8)]),
                                             ([5], [96])])
@pytest.mark.parametrize("n_parts", [1, 2, 3, 8])
def test_plan_tiles_partition_exact(class_n, class_w, n_parts):
    from paper_1102_1003_b200 import plan_tiles

    seen = []
    works = []
    for part in range(n_parts):
        tiles, work = plan_tiles(class_n, class_w, part, n_parts)
        seen.extend(map(tuple, tiles.tolist()))
        works.append(work)
        assert work == sum(128 * 128 * class_w[t[1]] for t in tiles.tolist())
    assert len(seen) == len(set(seen))
    assert set(seen) == _all_tiles(class_n, 128)
    # round-robin over cost-sorted tiles: parts differ by at most one (largest) tile
    biggest = 128 * 128 * max(class_w)
    assert max(works) - min(works) <= biggest


def test_plan_tiles_covers_every_pair_once():
    """Tiles (a<=b, diagonal tiles upper-triangular) cover each unordered pair exactly once."""
    from paper_1102_1003_b200 import plan_tiles

    class_n = [37, 20, 5]
    first = np.cumsum([0] + class_n)
    tiles, _ = plan_tiles(class_n, [96, 192, 384], 0, 1, tile_m=16)
    cover = {}
    for a, b, i, j in tiles.tolist():
        for r in range(i * 16, min(class_n[a], i * 16 + 16)):
            for c in range(j * 16, min(class_n[b], j * 16 + 16)):
                if a == b and r >= c:
                    continue
                key = (first[a] + r, first[b] + c)
                cover[key] = cover.get(key, 0) + 1
    n = sum(class_n)
    assert len(cover) == n * (n - 1) // 2 and set(cover.values()) == {1}
