"""Host-side checks of the C-ABI library (no GPU needed): it loads and exports
every entry point include/hg.h declares, and host-side validation rejects bad
sizes synchronously with HG_ERR_INVALID before touching the device."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "hg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hg_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_1908_08281_b200 import build
    lib_path = build.build()
    lib = ctypes.CDLL(lib_path)
    names = declared_symbols()
    assert len(names) >= 10
    for n in names:
        assert hasattr(lib, n), f"{n} declared in include/hg.h but not exported"
    from paper_1908_08281_b200 import hg
    assert set(hg.EXPORTS) == set(names)


def test_ragged_T_is_accepted():
    """T % 4 != 0 is valid (Y, F pass through 16-byte-pitched workspace copies), and costs more workspace."""
    from paper_1908_08281_b200 import hg
    assert hg.workspace_size(128, 10, 10, 64, 8, 7) > hg.workspace_size(128, 10, 10, 64, 8, 8)


def test_host_validation_is_synchronous_and_invalid():
    from paper_1908_08281_b200 import hg
    with pytest.raises(hg.HGError) as e:
        hg.workspace_size(100, 10, 10, 30, 8, 0)        # N % b != 0
    assert e.value.status == hg.HG_ERR_INVALID and "N % b" in str(e.value)
    for args in [(128, 10, 10, 64, 72, 0),                 # k > b
                 (128, 10, 10, 64, 6, 0),                  # k % 4
                 (128, 10, 10, 64, 8, -1),                 # T < 0
                 (1024, 10, 10, 1024, 1024, 0)]:           # k > 512
        with pytest.raises(hg.HGError) as e:
            hg.workspace_size(*args)
        assert e.value.status == hg.HG_ERR_INVALID
    assert hg.workspace_size(512, 548, 4937, 128, 32, 20) > 0


def test_workspace_grows_with_sizes():
    from paper_1908_08281_b200 import hg
    a = hg.workspace_size(4096, 4396, 62223, 256, 64, 100)
    b = hg.workspace_size(4096, 4396, 62223, 256, 128, 100)
    c = hg.workspace_size(8192, 4396, 62223, 256, 64, 100)
    assert b > a and c > a


def test_cg_host_validation():
    from paper_1908_08281_b200 import hg
    for args in [(512, 548, 4937, 6, 10),        # T % 4
                 (512, 548, 4937, 0, 10),        # T = 0
                 (512, 548, 4937, 20, -1),       # max_iter < 0
                 (0, 548, 4937, 20, 10)]:        # N = 0
        with pytest.raises(hg.HGError) as e:
            hg.cg_workspace_size(*args)
        assert e.value.status == hg.HG_ERR_INVALID
    a = hg.cg_workspace_size(512, 548, 4937, 20, 10)
    b = hg.cg_workspace_size(512, 548, 4937, 200, 10)
    assert 0 < a < b


def test_bounds_checked_build_has_the_checks():
    """libhgrsvd_check.so (HG_LIB=check, the compute-sanitizer substitute) carries the HG_DCHECK traps."""
    import shutil
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    counts = []
    for name in ("libhgrsvd.so", "libhgrsvd_check.so"):
        path = os.path.join(root, "paper_1908_08281_b200", name)
        assert os.path.exists(path), path
        sass = subprocess.run([cuobjdump, "-sass", path], capture_output=True, text=True).stdout
        counts.append(sass.count("BPT.TRAP"))
    assert counts[1] > counts[0] + 20, counts
