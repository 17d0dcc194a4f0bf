"""CPU-side checks of the C ABI library: it builds for sm_100a, loads, exports every symbol include/svg2.h declares,
validates arguments synchronously, and reports consistent workspace sizes.  No kernel is launched here."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2505_18875_b200 import build
    build.build()
    import paper_2505_18875_b200 as m
    return m.load_library()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "svg2.h")).read()
    return sorted(set(re.findall(r"\b(svg2_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_entry_points():
    names = declared_symbols()
    for n in ["svg2_kmeans", "svg2_permute", "svg2_select_topp", "svg2_varblock_attention", "svg2_unpermute",
              "svg2_sparse_attention"]:
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), f"libsvg2.so does not export {name}"


def test_binding_names_match_abi():
    import paper_2505_18875_b200 as m
    for n in ["kmeans", "permute", "select_topp", "varblock_attention", "unpermute", "sparse_attention"]:
        assert callable(getattr(m, n))
    assert sorted(m.EXPORTED_SYMBOLS) == sorted(declared_symbols())


def test_status_strings_and_version(lib):
    assert lib.svg2_abi_version() == 3
    assert lib.svg2_status_string(0) == b"SVG2_OK"
    assert lib.svg2_status_string(5) == b"SVG2_ERR_WORKSPACE_TOO_SMALL"


def test_workspace_sizes(lib):
    import paper_2505_18875_b200 as m
    ws = m.workspace_size(m.ENTRY_SPARSE_ATTENTION, 1, 24, 118800, 118800, 128, 100, 500, 2, 0.9)
    # Q', K', V' alone are 3 x 730 MB at the HunyuanVideo shape
    assert ws > 3 * 24 * 118800 * 128 * 2
    assert ws < 8 * 2**30
    assert m.workspace_size(m.ENTRY_SPARSE_ATTENTION, 1, 1, 100, 100, 128, 200, 5) == 0  # C > N -> invalid
    assert m.workspace_size(m.ENTRY_SPARSE_ATTENTION, 1, 1, 100, 100, 48, 2, 5) == 0  # d = 48 unsupported
    assert m.workspace_size(m.ENTRY_SELECT_TOPP, 1, 1, 100, 100, 128, 10, 10) >= 10 * 10 * 8  # fp64 score table
    assert m.workspace_size(m.ENTRY_SELECT_TOPP, 1, 1, 100, 100, 128, 10, 5000) == 0  # Ck > 4096


def test_validation_rejects_before_touching_the_device(lib):
    import paper_2505_18875_b200 as m
    cfg = m.Config(8, 8, 1, 0.9, 0.0, 0)
    dims = m.Dims(1, 1, 256, 256, 64)
    fake = ctypes.c_void_p(0x10000)
    # NULL workspace / outputs -> SVG2_ERR_NULL_POINTER
    assert lib.svg2_sparse_attention(fake, fake, fake, dims, ctypes.byref(cfg), fake, fake, fake, None, None, None,
                                     0, None) == 1
    # bad top_p -> SVG2_ERR_INVALID_PARAM (validated before any CUDA call)
    cfg_bad = m.Config(8, 8, 1, 0.0, 0.0, 0)
    assert lib.svg2_sparse_attention(fake, fake, fake, dims, ctypes.byref(cfg_bad), fake, fake, fake, None, None,
                                     fake, 1 << 30, None) == 3
    # misaligned pointer -> SVG2_ERR_MISALIGNED
    odd = ctypes.c_void_p(0x10008)
    assert lib.svg2_sparse_attention(odd, fake, fake, dims, ctypes.byref(cfg), fake, fake, fake, None, None, fake,
                                     1 << 30, None) == 4
    # too-small workspace -> SVG2_ERR_WORKSPACE_TOO_SMALL
    assert lib.svg2_sparse_attention(fake, fake, fake, dims, ctypes.byref(cfg), fake, fake, fake, None, None, fake,
                                     16, None) == 5
    # unknown flag bits -> SVG2_ERR_INVALID_PARAM; the k-means++ cold-start flag is accepted (then the fake pointers
    # fail the device check or later, never the parameter check)
    cfg_flag = m.Config(8, 8, 1, 0.9, 0.0, 8)
    assert lib.svg2_sparse_attention(fake, fake, fake, dims, ctypes.byref(cfg_flag), fake, fake, fake, None, None,
                                     fake, 1 << 30, None) == 3
    cfg_pp = m.Config(8, 8, 1, 0.9, 0.0, m.SVG2_INIT_KMEANSPP, 7)
    assert lib.svg2_sparse_attention(fake, fake, fake, dims, ctypes.byref(cfg_pp), fake, fake, fake, None, None,
                                     fake, 1 << 30, None) not in (1, 2, 3, 4, 5)
    # the FP8 PV path needs d = 128
    cfg_fp8 = m.Config(8, 8, 1, 0.9, 0.0, m.SVG2_FP8_PV)
    assert lib.svg2_sparse_attention(fake, fake, fake, dims, ctypes.byref(cfg_fp8), fake, fake, fake, None, None,
                                     fake, 1 << 30, None) == 3
    # svg2_kmeans: role must be 0 (queries) or 1 (keys)
    assert lib.svg2_kmeans(fake, 1, 1, 256, 64, 8, 1, m.SVG2_INIT_KMEANSPP, 7, 2, fake, fake, fake, None, None, None,
                           fake, 1 << 30, None) == 3
    # d unsupported -> SVG2_ERR_INVALID_SHAPE
    assert lib.svg2_sparse_attention(fake, fake, fake, m.Dims(1, 1, 256, 256, 80), ctypes.byref(cfg), fake, fake,
                                     fake, None, None, fake, 1 << 30, None) == 2


def test_layout_validation(lib):
    """svg2_sparse_attention_layout rejects bad layouts synchronously (before any device call): strides that are not
    positive multiples of 8 elements or shorter than a row, more than 16 output shards, shards that do not cover Nq,
    a NULL shard pointer, a misaligned shard, bad query-cluster part ranges, and an aux stream without its events."""
    import paper_2505_18875_b200 as m
    cfg = m.Config(8, 8, 1, 0.9, 0.0, 0)
    dims = m.Dims(1, 2, 256, 256, 64)
    fake = ctypes.c_void_p(0x10000)

    def call(lay, O=fake):
        return lib.svg2_sparse_attention_layout(fake, fake, fake, dims, ctypes.byref(cfg), ctypes.byref(lay), fake,
                                                fake, O, None, None, None, fake, 1 << 30, None)

    def layout(**kw):
        lay = m.Layout()
        for k, v in kw.items():
            if k.endswith("strides"):
                getattr(lay, k)[:] = v
            else:
                setattr(lay, k, v)
        return lay

    assert call(layout(q_strides=(256 * 2 * 64, 64, 2 * 64 + 4))) == 2  # sN not a multiple of 8
    assert call(layout(k_strides=(256 * 2 * 64, 64, 32))) == 2           # sN < d
    assert call(layout(v_strides=(0, 64, 128))) == 2                     # partly zero
    assert call(layout(part_begin=0, part_end=3, part_count=2)) == 3     # end > count
    assert call(layout(part_begin=1, part_end=1, part_count=2)) == 3     # empty range
    assert call(layout(part_begin=0, part_end=1, part_count=5000)) == 3  # count > 4096
    shards = (ctypes.c_void_p * 17)(*([0x10000] * 17))
    too_many = layout(o_shards=ctypes.cast(shards, ctypes.c_void_p), n_shards=17, shard_tokens=16,
                      o_strides=(16 * 2 * 64, 64, 128))
    assert call(too_many, O=None) == 2
    short = layout(o_shards=ctypes.cast(shards, ctypes.c_void_p), n_shards=2, shard_tokens=100,
                   o_strides=(100 * 2 * 64, 64, 128))
    assert call(short, O=None) == 2                                       # 2 x 100 < 256 tokens
    nulls = (ctypes.c_void_p * 2)(0x10000, None)
    with_null = layout(o_shards=ctypes.cast(nulls, ctypes.c_void_p), n_shards=2, shard_tokens=128,
                       o_strides=(128 * 2 * 64, 64, 128))
    assert call(with_null, O=None) == 1
    odd = (ctypes.c_void_p * 2)(0x10000, 0x10008)
    misaligned = layout(o_shards=ctypes.cast(odd, ctypes.c_void_p), n_shards=2, shard_tokens=128,
                        o_strides=(128 * 2 * 64, 64, 128))
    assert call(misaligned, O=None) == 4
    assert call(layout(aux_stream=0x1234)) == 1                           # aux stream without its events
    # a valid layout passes validation (then fails later on the fake pointers, never with a layout status)
    ok = layout(q_strides=(256 * 2 * 64, 64, 128), part_begin=0, part_end=1, part_count=2)
    assert call(ok) not in (1, 2, 3, 4, 5)


def test_sass_has_tcgen05_and_tma(lib):
    """The attention and the permutation path compile to Blackwell-native instructions (UTCHMMA, UTMALDG, LDTM)."""
    import subprocess
    from paper_2505_18875_b200 import build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", build.LIB], capture_output=True, text=True).stdout
    assert "UTCHMMA" in out and "UTMALDG" in out and "LDTM" in out and "STTM" in out


def test_product_does_not_import_oracle():
    """The product path never reaches the oracle (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2505_18875_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src and "svg2_oracle" not in src, f
