"""CPU-side checks of the product library: it builds, loads, exports every symbol the header declares,
its host logic (spec grammar / allocation / packed layout) matches the oracle, and -- with no GPU in
this container -- every compute entry point fails loudly instead of falling back."""
import ctypes as C

import numpy as np
import pytest

import paper_1812_09162_b200 as qb
from paper_1812_09162_b200 import _lib
from paper_1812_09162_b200.synth import random_codes


@pytest.fixture(scope="module")
def L():
    qb.build()
    return qb.lib()


def test_exports_every_declared_symbol(L):
    names = _lib.exported_symbols_declared_in_header()
    assert len(names) >= 18
    for n in names:
        assert hasattr(L, n), f"{n} is declared in include/qadc.h but not exported"


def test_spec_matches_oracle(L, port):
    for dims, text in [(128, "16x{4,4}"), (96, "12x{6,5,5}"), (128, "12x{6,5,5}"), (128, "12x{6,6,4}"),
                       (120, "12x{5,5,5}"), (128, "8x{8,8}"), (128, "8x{8}"), (64, "4x{4,4,4,4}"), (17, "2x{3,5}")]:
        assert bytes(qb.allocate_dims(dims, text)) == bytes(port.spec(dims, text)), text


@pytest.mark.parametrize("bad", ["x{4,4}", "16x{4,4", "16x{}", "16x{9}", "16x{4,}", "5x{4,4}", "16x{4,3}", "0x{8}",
                                 "16y{4,4}", "16x{4;4}"])
def test_bad_specs_are_invalid_spec_errors(L, bad):
    with pytest.raises(qb.QadcError) as e:
        qb.allocate_dims(128, bad)
    assert e.value.kind == "invalid_spec"


def test_too_few_dims(L):
    with pytest.raises(qb.QadcError) as e:
        qb.allocate_dims(8, "16x{4,4}")
    assert e.value.kind == "invalid_spec"


def test_host_layout_matches_oracle(L, port):
    for dims, text in [(128, "16x{4,4}"), (96, "12x{6,5,5}"), (128, "8x{8,8}"), (128, "8x{8}"), (24, "3x{5,5,5}")]:
        s, so = qb.allocate_dims(dims, text), port.spec(dims, text)
        for n in (0, 1, 15, 16, 17, 100, 1000):
            codes = random_codes(s, n, seed=n)
            pk = qb.pack_list(s, codes)
            assert pk.size == qb.packed_bytes(s, n) == port.packed_bytes(so, n)
            assert np.array_equal(pk, port.pack_list(so, codes))
            assert np.array_equal(qb.unpack_list(s, pk, n), codes)


def test_pack_overflow_is_corruption(L):
    s = qb.allocate_dims(8, "2x{4,4}")
    with pytest.raises(qb.QadcError) as e:
        qb.pack_list(s, np.array([[0x10, 3]], np.uint8))
    assert e.value.kind == "corruption"


def test_no_cpu_fallback(L):
    """Without a CUDA device the product must refuse to compute (status class 'cuda'), not emulate."""
    if L.qadc_device_count() > 0:
        pytest.skip("a GPU is visible; the fallback check only makes sense on a CPU box")
    s = qb.allocate_dims(64, "16x{4,4}")
    cb = np.zeros(s.cb_floats, np.float32)
    pk = qb.pack_list(s, np.zeros((4, 16), np.uint8))
    with pytest.raises(qb.QadcError) as e:
        qb.FlatIndex(s, cb, pk, 4)
    assert e.value.kind == "cuda"
    with pytest.raises(qb.QadcError) as e:
        qb.scan_list(s, pk, 4, np.zeros(256, np.uint8))
    assert e.value.kind == "cuda"
    with pytest.raises(qb.QadcError) as e:
        qb.encode(s, cb, np.zeros((2, 64), np.float32))
    assert e.value.kind == "cuda"


def test_product_does_not_link_the_oracle(L):
    import subprocess
    out = subprocess.run(["ldd", str(_lib.SO_PATH)], capture_output=True, text=True).stdout
    assert "oracle" not in out and "pqscan" not in out
    syms = subprocess.run(["nm", "-D", str(_lib.SO_PATH)], capture_output=True, text=True).stdout
    assert " orc_" not in syms


def test_cpp_binding_fails_loudly_without_gpu(L):
    """The reference-side C++ binding (include/qadc.hpp) must surface the missing device as an error, not emulate."""
    import subprocess
    from pathlib import Path
    if L.qadc_device_count() > 0:
        pytest.skip("a GPU is visible")
    exe = Path(__file__).resolve().parent.parent / "oracle" / "_ref" / "integration_test"
    if not exe.exists():
        pytest.skip("integration binary not built")
    out = subprocess.run([str(exe), "1"], capture_output=True, text=True, timeout=120)
    assert out.returncode != 0
    assert "no usable CUDA device" in out.stderr


# ------------------------------------------------ N1: container loader, host-side parsing --

def _open_raises(path):
    import ctypes as C
    h = C.c_void_p()
    rc = qb.lib().qadc_open_file(str(path).encode(), 0, C.byref(h))
    return rc, qb.lib().qadc_last_error().decode()


def test_container_parse_errors(L, tmp_path):
    """Header parsing mirrors io.hpp's error classes and happens before any device work (so it is testable here)."""
    from pathlib import Path
    gold = Path(__file__).resolve().parent / "golden"
    good = (gold / "flat_pq16x4.qflt").read_bytes()
    assert _open_raises(tmp_path / "missing.qflt")[0] == 8                      # io_error: cannot open
    p = tmp_path / "x.bin"
    p.write_bytes(b"NOPE" + good[4:])
    assert _open_raises(p)[0] == 8                                              # bad magic (io.hpp:54-58)
    p.write_bytes(good[:4] + (2).to_bytes(4, "little") + good[8:])
    assert _open_raises(p)[0] == 8                                              # unsupported version (io.hpp:288-289)
    p.write_bytes(good[: len(good) // 2])
    assert _open_raises(p)[0] == 8                                              # truncated (io.hpp:39)
    # QFLT(8) QADC(8) dims ngroups g widths(2) dim_alloc(16*4) codebook ... ; corrupt one dim_alloc entry
    off = 8 + 8 + 12 + 2
    bad = bytearray(good)
    bad[off] ^= 1
    p.write_bytes(bytes(bad))
    assert _open_raises(p)[0] == 6                                              # allocation mismatch (io.hpp:191-192)
    # flip a bit of the stored spec hash inside the QPKD header
    q = good.index(b"QPKD")
    bad = bytearray(good)
    bad[q + 8] ^= 0x40
    p.write_bytes(bytes(bad))
    rc, msg = _open_raises(p)
    assert rc == 6 and "hash" in msg                                            # io.hpp:258-259
    bad = bytearray(good)
    bad[q + 16] = 16                                                            # word width 8 -> 16
    p.write_bytes(bytes(bad))
    assert _open_raises(p)[0] == 6                                              # scheme mismatch (io.hpp:260-262)
    bad = bytearray(good)
    bad[q + 24] = 2                                                             # two lists in a flat index
    p.write_bytes(bytes(bad))
    assert _open_raises(p)[0] in (6, 8)                                         # io.hpp:293 (or EOF while reading list 2)
    if L.qadc_device_count() <= 0:
        assert _open_raises(gold / "flat_pq16x4.qflt")[0] == 20                 # a valid file still needs a device
