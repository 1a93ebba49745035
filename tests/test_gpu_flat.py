"""K0 (bind-time buffer packaging) on a real torch model: FlatParams gathers
every parameter into the flat fp32 bucket with the C-ABI gather kernel and re-points
parameters and grads as views that keep their memory format, so backward writes
straight into the gradient bucket and the DASO step updates the model in place."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import paper_2104_05588_b200 as daso  # noqa: E402


def small_cnn():
    torch.manual_seed(0)
    return torch.nn.Sequential(torch.nn.Conv2d(3, 16, 3), torch.nn.BatchNorm2d(16), torch.nn.ReLU(),
                               torch.nn.Conv2d(16, 8, 3), torch.nn.Flatten(), torch.nn.Linear(8 * 4 * 4, 10))


@pytest.mark.parametrize("channels_last", [False, True])
def test_flat_params_views_and_grads(channels_last):
    m = small_cnn().cuda()
    if channels_last:
        m = m.to(memory_format=torch.channels_last)
    before = [p.detach().clone() for p in m.parameters()]
    strides = [p.stride() for p in m.parameters()]
    flat = daso.FlatParams(m.parameters(), gpus_per_node=2)
    assert flat.n == sum((p.numel() + 63) // 64 * 64 for p in m.parameters())
    assert flat.n_pad % 128 == 0
    for p, b, st in zip(m.parameters(), before, strides):
        assert torch.equal(p.detach(), b) and p.stride() == st
        assert p.data_ptr() >= flat.x.data_ptr() and p.data_ptr() < flat.x.data_ptr() + 4 * flat.n_pad
    x = torch.randn(4, 3, 8, 8, device="cuda")
    if channels_last:
        x = x.to(memory_format=torch.channels_last)
    m(x).square().mean().backward()
    ref = small_cnn().cuda()
    if channels_last:
        ref = ref.to(memory_format=torch.channels_last)
    ref(x).square().mean().backward()
    for p, q, o in zip(m.parameters(), ref.parameters(), flat.offsets):
        torch.testing.assert_close(p.grad, q.grad, rtol=1e-5, atol=1e-6)
        assert p.grad.data_ptr() == flat.g.data_ptr() + 4 * o


def test_flat_params_step_updates_model_in_place():
    m = small_cnn().cuda()
    flat = daso.FlatParams(m.parameters())
    ctx = daso.daso_init(1, 1, 4, 1, rank=0, uid=daso.daso_get_unique_id(), wire="fp32")
    ctx.bind(flat.x, flat.g, flat.v, flat.n)
    w0 = m[0].weight.detach().clone()
    flat.g.zero_()
    m(torch.randn(4, 3, 8, 8, device="cuda")).square().mean().backward()
    gw = m[0].weight.grad.detach().clone()
    ctx.step(0.1)
    torch.cuda.synchronize()
    expect = w0 - 0.1 * (gw + 1e-4 * w0)      # first momentum step: v = d
    torch.testing.assert_close(m[0].weight.detach(), expect, rtol=1e-6, atol=1e-7)
    ctx.finalize()
