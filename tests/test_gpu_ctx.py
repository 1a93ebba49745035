"""Context-level behaviour of the C ABI on one GPU: protocol and argument errors
(SPEC S:437-446 error classes), tracing counters, the host-buffer step
(daso_step_host) and the non-finite flag."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import paper_2104_05588_b200 as daso  # noqa: E402
from paper_2104_05588_b200 import _lib as L  # noqa: E402


def ctx1(**kw):
    return daso.daso_init(1, 1, 4, 1, rank=0, uid=daso.daso_get_unique_id(), steps_per_epoch=64, **kw)


def bufs(n=1000):
    return [torch.zeros(n, device="cuda") for _ in range(3)]


def test_protocol_errors():
    c = ctx1()
    with pytest.raises(daso.DasoError) as e:
        c.step(0.1)                                   # step before bind
    assert e.value.status == L.ERR_PROTOCOL
    x, g, v = bufs()
    c.bind(x, g, v)
    with pytest.raises(daso.DasoError) as e:
        c.bind(x, g, v)                               # bind twice
    assert e.value.status == L.ERR_PROTOCOL
    with pytest.raises(daso.DasoError) as e:
        c.global_merge()                              # nothing in flight
    assert e.value.status == L.ERR_PROTOCOL
    with pytest.raises(daso.DasoError) as e:
        c.global_send(3, 1)                           # group out of range (G = 1)
    assert e.value.status == L.ERR_RANGE
    c.finalize()


def test_split_api_requires_faithful_mode():
    c = ctx1(mode="sharded")
    x, g, v = bufs(daso.daso_padded_numel(1000, 1))
    c.bind(x, g, v, 1000)
    with pytest.raises(daso.DasoError) as e:
        c.local_sync()
    assert e.value.status == L.ERR_PROTOCOL
    c.finalize()


def test_bind_argument_errors():
    c = ctx1()
    x = torch.zeros(1001, device="cuda")
    with pytest.raises(daso.DasoError) as e:
        c.bind(x[1:], x[1:].clone(), x[1:].clone())   # x misaligned (4-byte offset)
    assert e.value.status == L.ERR_ARGUMENT
    c.finalize()


def test_trace_counts_and_bytes():
    c = ctx1()
    n = 4096
    x, g, v = bufs(n)
    c.bind(x, g, v)
    c.trace_enable(True)
    for _ in range(8):
        c.step(0.1)
    t = c.trace_read()
    assert t["steps"] == 8 and t["kernel_launches"] == 8
    assert t["kernel_bytes"] == 8 * 20 * n            # K1 at 1x1: 20 B/param
    assert t["kernel_nvl_bytes"] == 0                  # no node tier at G = 1
    assert t["kernel_ms"] > 0 and t["local_ops"] == 0 and t["exch_ops"] == 0
    c.finalize()


def test_step_host_and_nonfinite_flag():
    c = ctx1(wire="fp32")
    n = 4096
    x, g, v = bufs(n)
    c.bind(x, g, v)
    hg = torch.ones(n, dtype=torch.float32).pin_memory()
    r, flag = c.step_host(hg, 0.5)
    assert flag == 0 and r["step"] == 0
    torch.testing.assert_close(x, torch.full_like(x, -0.5))     # x = 0 - 0.5 * (1 + 0)
    hg[7] = float("nan")
    _, flag = c.step_host(hg, 0.5)
    assert flag == 1
    assert c.check_finite()                                     # step_host already read and cleared it
    g.fill_(float("inf"))
    c.step(0.1)
    assert not c.check_finite()
    c.finalize()


def test_kernel_impl_switch_round_trips():
    prev = daso.daso_kernel_impl("tma")
    assert daso.daso_kernel_impl() == 1
    daso.daso_kernel_impl(prev)
    assert daso.daso_kernel_impl() == prev
