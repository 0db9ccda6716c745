"""C-ABI library checks that need no GPU: it loads, it exports every symbol
include/iccl_b200.h declares, and its host arithmetic (the product's own
SPEC formulas) agrees with the oracle."""
import ctypes as C
import os
import re
import subprocess
import sys

import pytest
from hypothesis import given, settings, strategies as st

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "iccl_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(iccl_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2510_00991_b200._lib import LIB_PATH, PROTOTYPES
    lib = C.CDLL(LIB_PATH)
    names = _header_functions()
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(PROTOTYPES), set(names) ^ set(PROTOTYPES)


def test_library_is_sm100a():
    from paper_2510_00991_b200._lib import LIB_PATH
    out = subprocess.run(["cuobjdump", "--list-elf", LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", LIB_PATH], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass  # K1's cp.async.bulk (TMA bulk copy)


def test_error_strings_and_version():
    from paper_2510_00991_b200._lib import lib
    assert lib.iccl_get_version() == 100
    assert lib.iccl_get_error_string(6) == b"ZeroLengthMessage"
    assert lib.iccl_get_error_string(12) == b"GroupTooSmall"


def test_no_gpu_init_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2510_00991_b200 import Communicator, IcclError
    with pytest.raises(Exception):
        Communicator(0, 1, 0)
    del IcclError


def test_retry_timeout_matches_oracle():
    from oracle.verbs import retry_timeout_ns
    from paper_2510_00991_b200._lib import lib
    for e in range(0, 20):
        for r in range(0, 8):
            assert lib.iccl_retry_timeout_ns(e, r) == retry_timeout_ns(e, r)
    from paper_2510_00991_b200 import retry_timeout
    assert retry_timeout(18, 7) == pytest.approx(8.589934592)  # G1


def test_switch_pointers_G14():
    from paper_2510_00991_b200._lib import XferState, lib
    s = XferState(posted=10, transmitted=9, acked=5)
    r = XferState(r_posted=10, received=8, done=6)
    assert lib.iccl_switch_pointers(C.byref(s), C.byref(r)) == 6
    assert (r.received, s.acked, s.transmitted, s.posted) == (6, 6, 6, 6)


@settings(max_examples=200, deadline=None)
@given(st.lists(st.tuples(st.integers(1, 1 << 26), st.integers(0, 10 ** 6), st.integers(1, 10 ** 6)),
                min_size=1, max_size=40), st.integers(1, 12))
def test_monitor_formulas_match_oracle(raw, window):
    from oracle import monitor as om
    from oracle.transport import MessageRecord as ORec
    import paper_2510_00991_b200 as p
    recs, orecs = [], []
    t = 0
    for i, (size, gap, dur) in enumerate(raw):
        t += gap
        recs.append(p.MessageRecord(size, t, t + dur))
        orecs.append(ORec(i, size, t, t + dur))
    got = p.sample_series(recs, window)
    exp = om.sample_series(orecs, window)
    assert len(got) == len(exp) == max(0, len(raw) - window + 1)
    for a, b in zip(got, exp):
        assert a.time == b.time
        assert a.value == pytest.approx(b.value, rel=1e-12)
    for r, o in zip(recs, orecs):
        assert p.per_message_throughput(r) == pytest.approx(om.per_message_throughput(o.size, o.t1, o.t2))


def test_monitor_errors():
    import paper_2510_00991_b200 as p
    R = p.MessageRecord
    with pytest.raises(p.NonPositiveDuration):
        p.per_message_throughput(R(1, 5, 5))
    with pytest.raises(p.WindowNotFull):
        p.window_throughput([R(1, 0, 10)] * 3, 4)
    assert p.window_throughput([R(1 << 20, 0, 100_000)] * 4, 4) == pytest.approx(41.94304e9)  # G20


@settings(max_examples=300, deadline=None)
@given(st.dictionaries(st.integers(0, 15), st.integers(0, 1000), min_size=2, max_size=16), st.integers(0, 5))
def test_lagging_rank_matches_oracle(counts, thr):
    from oracle.monitor import detect_lagging_rank as ref
    import paper_2510_00991_b200 as p
    assert p.detect_lagging_rank(counts, thr) == ref(counts, thr)


def test_config_defaults_and_env_override():
    import paper_2510_00991_b200 as p
    d = p.IcclConfig.defaults()
    assert d.monitor_window == 8 and d.timeout_exponent == 18 and d.retry_count == 7  # Table 5
    code = ("import paper_2510_00991_b200 as p; c=p.IcclConfig.defaults(); "
            "print(c.chunk_bytes, c.timeout_exponent, c.retry_count, c.monitor_window, c.transport)")
    env = dict(os.environ, ICCL_CHUNK_BYTES="8M", ICCL_IB_TIMEOUT="12", ICCL_IB_RETRY_CNT="3",
               ICCL_MONITOR_WINDOW="32", ICCL_TRANSPORT="2")
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=ROOT, capture_output=True, text=True)
    assert out.stdout.split() == [str(8 << 20), "12", "3", "32", "sm"], out.stderr


def test_path_selection_defaults_and_overrides():
    """The size classes of the data path: LL (K5) <= 256 KiB < direct (K6)
    <= 16 MiB < copy engines; relay staging 32 MiB; each an ICCL_* knob."""
    import paper_2510_00991_b200 as p
    d = p.IcclConfig.defaults()
    assert (d.sm_small_bytes, d.direct_max_kib, d.relay_slot_mib, d.backup_kind) == (1024 * 1024, 16 * 1024, 32, "sm")
    code = ("import paper_2510_00991_b200 as p; c=p.IcclConfig.defaults(); "
            "print(c.sm_small_bytes, c.direct_max_kib, c.relay_slot_mib, c.backup_kind)")
    env = dict(os.environ, ICCL_SM_SMALL_BYTES="4096", ICCL_DIRECT_MAX_KIB="0", ICCL_RELAY_SLOT_MIB="8",
               ICCL_BACKUP="1")
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=ROOT, capture_output=True, text=True)
    assert out.stdout.split() == ["4096", "0", "8", "relay"], out.stderr
    with pytest.raises(p.InvalidConfig):
        p.IcclConfig.defaults(direct_max_kib=-1).validate()
    with pytest.raises(p.InvalidConfig):
        p.IcclConfig.defaults(relay_slot_mib=0).validate()


def test_config_validation():
    import paper_2510_00991_b200 as p
    with pytest.raises(p.InvalidConfig):
        p.IcclConfig.defaults(monitor_window=0).validate()
    with pytest.raises(p.InvalidConfig):
        p.IcclConfig.defaults(chunk_bytes=100).validate()
    with pytest.raises(p.ConfigError):
        p.IcclConfig.defaults(no_such_field=1)


def test_fault_script_validation():
    import paper_2510_00991_b200 as p
    fs = p.FaultScript().down(0, 1, t_us=10).up(0, 1, t_us=20)
    fs.validate(2)
    with pytest.raises(p.InvalidArgument):
        p.FaultScript().down(0, 5).validate(2)  # UnknownPort
    with pytest.raises(p.InvalidArgument):
        p.FaultScript().down(0, 1).down(0, 1).validate(2)  # Down/Up must alternate
    with pytest.raises(p.InvalidArgument):
        p.FaultScript().down(0, 1, t_us=30).up(0, 1, t_us=10).validate(2)  # time order


def test_unique_id_without_gpu():
    from paper_2510_00991_b200._lib import UniqueId, lib
    a, b = UniqueId(), UniqueId()
    assert lib.iccl_get_unique_id(C.byref(a)) == 0
    assert lib.iccl_get_unique_id(C.byref(b)) == 0
    assert bytes(a.internal) != bytes(b.internal)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2510_00991_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", txt, re.M), f
