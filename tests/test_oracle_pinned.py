"""The oracle itself is pinned before it is trusted:
  * the unmodified reference library passes the reference's own unit tests
    (35 cases, 103,739 checks) under oracle/doctest.h;
  * the C restatement of the byte functions (oracle/swap_oracle.c) matches
    splitmix64's published first output and is self-consistent."""
import ctypes
import os
import subprocess

import pytest

from conftest import REF_BIN


def test_reference_unit_tests_pass():
    exe = os.path.join(REF_BIN, "ref_unit_tests")
    if not os.path.exists(exe):
        pytest.skip("reference not built here (needs /root/reference at build time)")
    p = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    assert "test cases: 35 | 0 failed" in p.stdout and "failures: 0" in p.stdout, p.stdout


def test_splitmix64_known_answers(oracle_lib):
    # Published splitmix64 stream for state 0: first outputs.
    assert oracle_lib.so_splitmix64(0) == 0xE220A8397B1DCDAF
    assert oracle_lib.so_splitmix64(0x9E3779B97F4A7C15) == 0x6E789E6AA1B965F4
    assert oracle_lib.so_splitmix64(2 * 0x9E3779B97F4A7C15 & (2**64 - 1)) == 0x06C45D188009454F


def test_pattern_checksum_self_consistent(oracle_lib):
    buf = ctypes.create_string_buffer(2 << 20)
    for app, block in [(0, 0), (1, 77), (3, 12345)]:
        oracle_lib.so_fill_block(buf, 0x4E495849, app, block)
        words = (ctypes.c_uint64 * 4).from_buffer(buf)
        assert words[0] == oracle_lib.so_pattern_word(0x4E495849, app, block, 0)
        assert words[3] == oracle_lib.so_pattern_word(0x4E495849, app, block, 3)
        ck = oracle_lib.so_checksum(buf, (2 << 20) // 8)
        assert ck == oracle_lib.so_pattern_block_checksum(0x4E495849, app, block)
        assert oracle_lib.so_compare_block(buf, 0x4E495849, app, block) == 0
        raw = bytearray(buf.raw)
        raw[4097] ^= 0x40
        bad = ctypes.create_string_buffer(bytes(raw), len(raw))
        assert oracle_lib.so_compare_block(bad, 0x4E495849, app, block) == 1
        assert oracle_lib.so_checksum(bad, (2 << 20) // 8) != ck


def test_checksum_detects_swapped_words(oracle_lib):
    buf = ctypes.create_string_buffer(2 << 20)
    oracle_lib.so_fill_block(buf, 5, 0, 1)
    ck = oracle_lib.so_checksum(buf, (2 << 20) // 8)
    w = (ctypes.c_uint64 * 16).from_buffer(buf)
    w[3], w[9] = w[9], w[3]
    assert oracle_lib.so_checksum(buf, (2 << 20) // 8) != ck
