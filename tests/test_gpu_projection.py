"""P1 decode-size projections (kvs_proj_skinny: the projection GEMMs of
decode steps, model.py:193-195 and :202) against a plain PyTorch fp32
reference of the same op: the three benched widths (Llama/Yi 4096, Qwen
3584), every row-count class (1..64, ragged), the bf16 QKV output and the
fp32 residual accumulate with its bf16 operand copy; repeat launches are
bit-identical (fixed summation order); shape errors raise."""
import pytest
import torch

from paper_2503_16525_b200 import _native as N
from paper_2503_16525_b200.engine import Engine
from paper_2503_16525_b200.errors import KVLabError

pytestmark = pytest.mark.gpu

TOL = 1e-2          # bf16 output / bf16 operands with fp32 accumulation


def _case(m, k, n, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = (torch.randn(m, k, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    w = (torch.randn(k, n, device="cuda", generator=g) / k ** 0.5).to(torch.bfloat16)
    return x, w, Engine.pack_skinny(w)


def _skinny(x, w_p, out, accumulate, out_bf16=None):
    n, k = w_p.shape[0] * 16, w_p.shape[1] * 64
    N.call("kvs_proj_skinny", x.data_ptr(), x.shape[0], w_p.data_ptr(), n, k, accumulate,
           out.data_ptr(), N.ptr(out_bf16), N.stream_ptr())


@pytest.mark.parametrize("k,n", [(4096, 6144), (4096, 4096), (3584, 4608), (3584, 3584),
                                 (4096, 5120)])
@pytest.mark.parametrize("m", [1, 5, 8, 13, 16, 32, 40, 64])
def test_qkv_output_matches_fp32(m, k, n):
    x, w, w_p = _case(m, k, n, seed=m * 7 + n)
    out = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
    _skinny(x, w_p, out, 0)
    ref = x.float() @ w.float()
    err = (out.float() - ref).abs().max().item()
    assert err <= TOL * ref.abs().max().item(), err


@pytest.mark.parametrize("k,n", [(4096, 4096), (3584, 3584)])
@pytest.mark.parametrize("m", [3, 32, 64])
def test_residual_accumulate_and_operand_copy(m, k, n):
    x, w, w_p = _case(m, k, n, seed=m + k)
    res0 = torch.randn(m, n, device="cuda")
    res = res0.clone()
    xb = torch.zeros(m, n, dtype=torch.bfloat16, device="cuda")
    _skinny(x, w_p, res, 1, xb)
    ref = res0 + x.float() @ w.float()
    scale = ref.abs().max().item()
    assert (res - ref).abs().max().item() <= 1e-4 * scale + 1e-4
    assert torch.equal(xb, res.to(torch.bfloat16))          # bf16(x) for the next layer


def test_repeat_launches_bit_identical():
    x, w, w_p = _case(32, 4096, 6144, seed=3)
    a = torch.empty(32, 6144, dtype=torch.bfloat16, device="cuda")
    b = torch.empty_like(a)
    _skinny(x, w_p, a, 0)
    for _ in range(3):
        _skinny(x, w_p, b, 0)
        assert torch.equal(a, b)


def test_shape_errors_raise():
    x, w, w_p = _case(65, 4096, 4096, seed=1)
    out = torch.empty(65, 4096, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(KVLabError):
        _skinny(x, w_p, out, 0)                               # m > 64
    with pytest.raises(KVLabError):                           # k % 512 != 0
        N.call("kvs_proj_skinny", x.data_ptr(), 8, w_p.data_ptr(), 4096, 1000, 0,
               out.data_ptr(), None, N.stream_ptr())
    with pytest.raises(KVLabError):
        _skinny(x[:8], w_p, out, 0, out_bf16=out)             # out_bf16 without accumulate


def test_engine_routes_decode_rows_through_p1():
    """A Llama-width engine sends <= 64-row projections through P1; the
    results match the library GEMM path within the bf16 tolerance."""
    from paper_2503_16525_b200.engine import Engine
    from paper_2503_16525_b200.model import ModelConfig, init_model
    from paper_2503_16525_b200.pool import CachePool

    cfg = ModelConfig(num_layers=2, num_heads=32, d_model=4096, vocab_size=512, num_kv_heads=8)
    model = init_model(cfg, device="cuda")
    eng = Engine(model, CachePool(cfg, arena_pages=8))
    x = torch.randn(24, 4096, device="cuda")
    o = (torch.randn(24, 32, 128, device="cuda") * 0.3).to(torch.bfloat16)
    outs = []
    for skinny in (True, False):
        eng.skinny, eng._xb_of = skinny, None
        xs = x.clone()
        qkv = eng._qkv(xs, 1).clone()
        eng._out_proj(xs, o, 1)
        outs.append((qkv, xs))
    assert eng._wt is not None
    (q1, x1), (q2, x2) = outs
    assert (q1.float() - q2.float()).abs().max().item() <= TOL * q2.float().abs().max().item()
    assert (x1 - x2).abs().max().item() <= 1e-4 * x2.abs().max().item() + 1e-3
