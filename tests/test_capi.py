"""CPU: the C-ABI library loads, exports every symbol include/ros_b200.h
declares, and its host-only entry points behave without a GPU."""
import ctypes as C
import os
import re

import pytest

from tests.conftest import ROOT


def header_symbols():
    text = open(os.path.join(ROOT, "include", "ros_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\*]+\s+)+\*?(rs_\w+)\(", text, re.M)))


def test_header_declares_the_ros_surface():
    syms = header_symbols()
    for s in ("rs_open", "rs_register", "rs_publish", "rs_unpublish", "rs_replicate", "rs_update",
              "rs_locate", "rs_close", "rs_serve_export", "rs_serve_import"):
        assert s in syms
    assert len(syms) >= 45


def test_library_exports_every_declared_symbol():
    from paper_2604_09107_b200 import _lib
    for s in header_symbols():
        assert hasattr(_lib.lib, s), s
    assert set(header_symbols()) == set(_lib.EXPORTED)


def test_abi_and_status_names():
    from paper_2604_09107_b200._lib import lib
    from paper_2604_09107_b200.ros import Status
    assert lib.rs_abi_version() == 3
    for s in Status:
        assert lib.rs_status_name(int(s)).decode() == s.name  # types.cpp:7-29
    assert lib.rs_status_name(99).decode() == "unknown"


def test_config_defaults_mirror_reference():
    from paper_2604_09107_b200._lib import RsConfig, lib
    c = RsConfig()
    lib.rs_config_default(C.byref(c))
    assert c.tiny_threshold == 2 << 20 and c.group_target == 64 << 20  # manifest.hpp:46-49
    assert c.checksum_retries == 3 and c.pull_timeout_s == 4.0 and c.pipeline == 1  # config.hpp
    assert c.datacenter == b"dc0"


def test_bad_arguments_fail_loudly_without_gpu():
    from paper_2604_09107_b200.ros import Cluster, Status
    with Cluster() as cl:
        h = cl.open("m", "R", 1)
        # host memory is not registrable (regions live in device memory)
        import numpy as np
        a = np.zeros(16, np.uint8)
        assert h.register_tensor(0, "x", ptr=a.ctypes.data, nbytes=16) == Status.invalid_argument
        assert h.register_tensor(0, "", ptr=a.ctypes.data, nbytes=16) == Status.invalid_argument
        # the reference rejects '|' in names and empty regions (client_core.cpp:537-540)
        assert h.register_tensor(0, "a|b", ptr=a.ctypes.data, nbytes=16) == Status.invalid_argument
        assert h.register_tensor(0, "x", ptr=a.ctypes.data, nbytes=0) == Status.invalid_argument
        assert h.register_tensor(1, "x", ptr=a.ctypes.data, nbytes=16) == Status.invalid_argument
        assert h.replicate("bogus").status == Status.invalid_argument
        # nothing registered: cannot open the replica
        assert h.publish(1).status == Status.invalid_state
        with pytest.raises(Exception):
            cl.locate("m", "nobody")
        # a closed handle refuses registrations (Status::closed)
        h.close()
        assert h.register_tensor(0, "y", ptr=a.ctypes.data, nbytes=16) in (Status.closed,
                                                                              Status.invalid_argument)
