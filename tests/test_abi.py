"""Host-side checks of the C-ABI library (no GPU needed, no compute calls).

- libhm.so loads and exports every function include/hm.h declares;
- the workspace queries follow the documented layout;
- invalid arguments are rejected on the host with the documented status and
  a message, before anything is launched.
"""
import ctypes
import os
import re
import subprocess

import pytest

import paper_1909_07909_b200 as hm
from paper_1909_07909_b200 import build as hm_build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    hm_build.build()
    return hm.load()


def header_functions():
    src = open(os.path.join(ROOT, "include", "hm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:hm_status|const char\*|int32_t)\s+(\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_binding_names():
    fns = header_functions()
    assert set(fns) == set(hm.EXPORTS), fns


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", hm.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [f for f in header_functions() if f not in exported]
    assert not missing, missing


def test_abi_version_and_no_error():
    lib = hm.load()
    assert lib.hm_abi_version() == 2
    assert isinstance(hm.hm_last_error(), str)


def test_library_has_no_torch_dependency():
    out = subprocess.run(["ldd", hm.LIB_PATH], capture_output=True, text=True).stdout
    # library names only: the load addresses ldd prints are random hex and can
    # contain "c10" (a flaky match before)
    names = [line.split()[0] for line in out.splitlines() if line.strip()]
    assert not [nm for nm in names if re.search(r"torch|c10", nm)], names


def test_kernels_are_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", hm.LIB_PATH], capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_hodlr_workspace_layout():
    n, p, b, k = 1 << 20, 12, 256, 16
    m = 8
    ws = hm.hm_hodlr_workspace_bytes(n, p, b, [k] * p, m)
    coef = sum((1 << l) * k * m * 8 for l in range(1, p + 1))
    assert ws >= coef
    assert ws < coef + 64 * 1024 * 1024  # partials stay small (tile-granular)
    ws_io = hm.hm_hodlr_workspace_bytes(n, p, b, [k] * p, m, hm.HM_WS_HOSTIO)
    assert ws_io >= ws + 2 * n * m * 8


def test_hss_workspace_layout():
    n, p, b, k, m = 1 << 22, 15, 128, 32, 32
    ws = hm.hm_hss_workspace_bytes(n, p, b, k, m)
    assert ws >= 2 * ((1 << (p + 1)) - 2) * k * m * 8


@pytest.mark.parametrize("n,levels,leaf,err", [
    (1000, 2, 256, hm.HM_ERR_UNSUPPORTED),   # not leaf * 2^levels (general tree)
    (0, 0, 1, hm.HM_ERR_INVALID_ARG),
    (1024, -1, 1024, hm.HM_ERR_INVALID_ARG),
])
def test_bad_trees_rejected(n, levels, leaf, err):
    with pytest.raises(hm.HmError) as e:
        hm.hm_hodlr_workspace_bytes(n, levels, leaf, [4] * max(levels, 0), 1)
    assert e.value.status == err
    assert len(hm.hm_last_error()) > 0


def test_bad_ranks_and_nrhs_rejected():
    with pytest.raises(hm.HmError) as e:
        hm.hm_hodlr_workspace_bytes(1024, 2, 256, [4, -1], 1)
    assert e.value.status == hm.HM_ERR_INVALID_ARG
    # per-level ranks run on the general-tree kernels
    assert hm.hm_hodlr_workspace_bytes(1024, 2, 256, [4, 8], 1) > 0
    with pytest.raises(hm.HmError) as e:
        hm.hm_hodlr_workspace_bytes(1024, 2, 256, [4, 65], 1)
    assert e.value.status == hm.HM_ERR_UNSUPPORTED
    with pytest.raises(hm.HmError) as e:
        hm.hm_hodlr_workspace_bytes(1024, 2, 256, [4, 4], 0)
    assert e.value.status == hm.HM_ERR_INVALID_ARG
    with pytest.raises(hm.HmError) as e:
        hm.hm_hss_workspace_bytes(1024, 2, 256, 65, 1)
    assert e.value.status == hm.HM_ERR_UNSUPPORTED


def test_matvec_validation_happens_before_launch():
    """Invalid calls return on the host (this container has no GPU, so reaching a launch
    would fail differently): NULL pointers, small workspace, overlapping X/Y."""
    lib = hm.load()
    t = hm.make_tree(1024, 2, 256)
    ranks = (ctypes.c_int32 * 2)(4, 4)
    buf = ctypes.create_string_buffer(1 << 16)
    base = (ctypes.addressof(buf) + 255) // 256 * 256
    rc = lib.hodlr_matvec(ctypes.byref(t), ranks, None, None, None, None, 1, None, base, 1 << 15, None)
    assert rc == hm.HM_ERR_INVALID_ARG or rc == hm.HM_ERR_WORKSPACE
    need = hm.hm_hodlr_workspace_bytes(1024, 2, 256, [4, 4], 1)
    rc = lib.hodlr_matvec(ctypes.byref(t), ranks, 16, 16, 16, 16, 1, 16, base, need - 1, None)
    assert rc == hm.HM_ERR_WORKSPACE
    # X and Y overlap
    rc = lib.hodlr_matvec(ctypes.byref(t), ranks, 256, 256, 256, 4096, 1, 4096 + 8, base, need, None)
    assert rc == hm.HM_ERR_INVALID_ARG and "overlap" in hm.hm_last_error()
    # misaligned D
    rc = lib.hodlr_matvec(ctypes.byref(t), ranks, 8, 256, 256, 4096, 1, 1 << 20, base, need, None)
    assert rc == hm.HM_ERR_INVALID_ARG and "aligned" in hm.hm_last_error()


def test_binding_refuses_cpu_tensors():
    torch = pytest.importorskip("torch")
    x = torch.zeros(1024, 1, dtype=torch.float64)
    with pytest.raises(TypeError):
        hm.hodlr_matvec(1024, 2, 256, [4, 4], x, x, x, x)


def test_general_tree_validation():
    """Endpoint vectors: nondecreasing, last = n; empty leaves allowed."""
    c = [3, 7, 7, 20, 26, 26, 31, 40]
    assert hm.hm_hodlr_general_workspace_bytes(40, 3, c, [2, 1, 3], 2) > 0
    assert hm.hm_hss_general_workspace_bytes(40, 3, c, 4, 2) > 0
    for bad, st in (([3, 7, 6, 20, 26, 26, 31, 40], hm.HM_ERR_INVALID_ARG),   # decreasing
                    ([3, 7, 7, 20, 26, 26, 31, 39], hm.HM_ERR_INVALID_ARG)):  # last != n
        with pytest.raises(hm.HmError) as e:
            hm.hm_hodlr_general_workspace_bytes(40, 3, bad, [2, 1, 3], 2)
        assert e.value.status == st
    with pytest.raises(hm.HmError) as e:  # one leaf larger than the shared-memory staging
        hm.hm_hss_general_workspace_bytes(30000, 1, [29000, 30000], 4, 1)
    assert e.value.status == hm.HM_ERR_UNSUPPORTED
    with pytest.raises(ValueError):
        hm.hm_hodlr_general_workspace_bytes(40, 3, c[:4], [2, 1, 3], 2)


def _build_c_example(tmp_path, name="hm_matvec_example"):
    """Compile examples/<name>.c (plain C, include/hm.h only) against libhm.so."""
    exe = str(tmp_path / name)
    libdir = os.path.dirname(hm.LIB_PATH)
    cuda_lib = "/usr/local/cuda/lib64"
    cmd = ["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "examples", name + ".c"), "-o", exe, "-L", libdir, "-l:libhm.so",
           "-L", cuda_lib, "-lcudart", f"-Wl,-rpath,{libdir}:{cuda_lib}", "-lm"]
    if name != "hm_matvec_example":
        cmd[1] = "-std=gnu99"  # fork / pipe
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_example_links_and_validates(tmp_path):
    """The C-ABI is usable from plain C: the example compiles against include/hm.h, links
    libhm.so, queries a workspace and sees an invalid tree rejected on the host."""
    exe = _build_c_example(tmp_path)
    out = subprocess.run([exe, "--host-only"], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0, out.stderr
    assert "invalid tree rejected" in out.stdout


def test_c_dist_example_links_host_only(tmp_path):
    """The distributed C-ABI from plain C: examples/hm_dist_example.c compiles against
    include/hm.h, queries the distributed workspaces, creates a communicator id (NCCL,
    loaded at run time) and sees P = 3 rejected — no GPU needed."""
    exe = _build_c_example(tmp_path, "hm_dist_example")
    out = subprocess.run([exe, "--host-only"], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "communicator id created" in out.stdout


def test_library_does_not_link_nccl():
    """NCCL is dlopen'ed by hm_comm_* only: the single-GPU calls load without it."""
    out = subprocess.run(["ldd", hm.LIB_PATH], capture_output=True, text=True).stdout
    assert "nccl" not in out


def test_comm_unique_id_on_host():
    from paper_1909_07909_b200 import dist as hd
    a, b = hd.unique_id(), hd.unique_id()
    assert len(a) == hd.HM_COMM_ID_BYTES and a != b


def test_dist_workspace_queries():
    from paper_1909_07909_b200 import dist as hd
    for P in (1, 2, 8):
        assert hd.hodlr_dist_workspace_bytes(1 << 16, 8, 256, [16] * 8, 8, P) > 0
        assert hd.hss_dist_workspace_bytes(1 << 15, 8, 128, 32, 32, P) > 0
    with pytest.raises(hm.HmError) as e:
        hd.hodlr_dist_workspace_bytes(1 << 16, 8, 256, [16] * 8, 8, 3)
    assert e.value.status == hm.HM_ERR_UNSUPPORTED
    with pytest.raises(hm.HmError):
        hd.hss_dist_workspace_bytes(1 << 15, 8, 128, 32, 32, 512)   # P > 2^levels


def test_struct_layouts_match_header(tmp_path):
    """The binding's ctypes records have the C header's sizes and field offsets
    (hm_tree, hm_part, hm_launch_record): a plain-C probe compiled against
    include/hm.h prints them."""
    import ctypes
    import subprocess
    import paper_1909_07909_b200 as hm
    from paper_1909_07909_b200 import dist
    recs = {
        "hm_tree": (hm.hm_tree, ["n", "levels", "flags", "leaf"]),
        "hm_part": (dist.hm_part, ["nranks", "rank"]),
        "hm_launch_record": (hm.hm_launch_record, ["name", "call", "ms", "start_ms"]),
    }
    src = ["#include <stdio.h>", "#include <stddef.h>", '#include "hm.h"', "int main(void) {"]
    for name, (_, fields) in recs.items():
        src.append(f'  printf("{name} %zu", sizeof({name}));')
        for f in fields:
            src.append(f'  printf(" %zu", offsetof({name}, {f}));')
        src.append('  printf("\\n");')
    src += ["  return 0;", "}"]
    c = tmp_path / "layout.c"
    c.write_text("\n".join(src) + "\n")
    exe = str(tmp_path / "layout")
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), str(c), "-o", exe],
                   check=True, capture_output=True, text=True)
    out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout.split("\n")
    for line in filter(None, out):
        name, size, *offs = line.split()
        cls, fields = recs[name]
        assert ctypes.sizeof(cls) == int(size), name
        assert [getattr(cls, f).offset for f in fields] == [int(o) for o in offs], name
