"""The memory model the planner uses (Eq. 6; reading R-22) against the
device: pds_mem_bytes' saved arena + workspace equals what the library actually
allocates (measured with cudaMemGetInfo around a forward), backward allocates
nothing more, and an allocation the device cannot satisfy surfaces as PDS_ENOMEM
and leaves the context usable.  This is the independent pin of the workspace term
(oracle/memory.py only bounds it below, by the dataflow floor)."""
import pytest
import torch

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2511_13198_b200 import binding as B

H, N, F = 4096, 32, 16384
MIB = 1 << 20


def _buffers(s, b=1):
    keys = ("w_qkv_t", "w_proj", "w_in_t", "w_out", "g1", "g2")
    shapes = dict(w_qkv_t=(3 * H, H), w_proj=(H, H), w_in_t=(F, H), w_out=(F, H), g1=(H,), g2=(H,))
    w = {k: (torch.randn(shapes[k], device="cuda") * 0.02).to(torch.bfloat16) for k in keys}
    g = {k: torch.zeros(shapes[k], device="cuda") for k in keys}
    x = torch.randn(s * b, H, device="cuda").to(torch.bfloat16)
    W = B.Weights(*(w[k].data_ptr() for k in keys))
    G = B.Grads(*(g[k].data_ptr() for k in keys))
    return w, g, x, W, G


def _free():
    torch.cuda.synchronize()
    return torch.cuda.mem_get_info()[0]


@pytest.mark.parametrize("pi", [0, 1, 2, 3, 4, 5])
def test_device_allocation_equals_mem_bytes(pi):
    s = 16384
    model = B.Model(h=H, n_heads=N, ffn=F, metp_chunks=4)
    w, g, x, W, G = _buffers(s)
    y, dx = torch.empty_like(x), torch.empty_like(x)
    st = torch.cuda.current_stream().cuda_stream
    ctx = B.Context(model)
    # warm-up at the same length: module loading, the RoPE table, streams and events
    sv = ctx.layer_fwd(pi, s, x.data_ptr(), W, y.data_ptr(), st)
    ctx.layer_bwd(pi, x.data_ptr(), sv, W, G, dx.data_ptr(), st)
    ctx.release_cache()
    f0 = _free()
    sv = ctx.layer_fwd(pi, s, x.data_ptr(), W, y.data_ptr(), st)
    f1 = _free()
    ctx.layer_bwd(pi, x.data_ptr(), sv, W, G, dx.data_ptr(), st)
    f2 = _free()
    saved, ws, _ = B.mem_bytes(model, 1, pi, s)
    x_bytes = s * H * 2                     # the retained input is the caller's buffer
    predicted = saved - x_bytes + ws
    used = f0 - f1
    # two cudaMalloc calls (saved arena, workspace), each rounded to 2 MiB pages
    assert 0 <= used - predicted <= 4 * MIB, (pi, used, predicted)
    assert f2 == f1, "backward must not allocate"
    ctx.close()


def test_enomem_is_reported_and_recoverable():
    s, pi = 16384, 0
    model = B.Model(h=H, n_heads=N, ffn=F)
    w, g, x, W, G = _buffers(s)
    y, dx = torch.empty_like(x), torch.empty_like(x)
    st = torch.cuda.current_stream().cuda_stream
    ctx = B.Context(model)
    sv = ctx.layer_fwd(pi, s, x.data_ptr(), W, y.data_ptr(), st)
    ctx.layer_bwd(pi, x.data_ptr(), sv, W, G, dx.data_ptr(), st)
    ctx.release_cache()
    saved, ws, _ = B.mem_bytes(model, 1, pi, s)
    need = saved - s * H * 2 + ws
    # leave 256 MiB less than the forward needs
    filler = torch.empty(_free() - need + 256 * MIB, dtype=torch.uint8, device="cuda")
    with pytest.raises(B.PdsError) as e:
        ctx.layer_fwd(pi, s, x.data_ptr(), W, y.data_ptr(), st)
    assert e.value.code == -4                                  # PDS_ENOMEM
    del filler
    torch.cuda.empty_cache()
    # the context recovers: the same call now runs and matches a fresh context bit for bit
    sv = ctx.layer_fwd(pi, s, x.data_ptr(), W, y.data_ptr(), st)
    ctx.layer_bwd(pi, x.data_ptr(), sv, W, G, dx.data_ptr(), st)
    y2, dx2 = torch.empty_like(x), torch.empty_like(x)
    ctx2 = B.Context(model)
    sv = ctx2.layer_fwd(pi, s, x.data_ptr(), W, y2.data_ptr(), st)
    ctx2.layer_bwd(pi, x.data_ptr(), sv, W, G, dx2.data_ptr(), st)
    torch.cuda.synchronize()
    assert torch.equal(y, y2) and torch.equal(dx, dx2)
    ctx.close()
    ctx2.close()
