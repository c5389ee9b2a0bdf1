"""The fused head kernel (head_fused.cu: a4 loss + the head's a5 in one launch) against the
oracle (C-T3 / C-T4) and against the three-kernel head path (SRL_HEAD_FUSED=0) it replaces,
on ragged row counts (n < 128, n % 128 != 0) and on sizes where every CTA takes several tiles
(the TMEM-resident dW_h accumulation across tiles)."""
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from ppo_harness import gpu_step, grad_errors, make_inputs, tensor_slices

pytestmark = pytest.mark.gpu
TOL = 2e-3


def _run(cfg, params, b, fused, apply=False):
    old = os.environ.get("SRL_HEAD_FUSED")
    os.environ["SRL_HEAD_FUSED"] = "1" if fused else "0"
    try:
        return gpu_step(cfg, params, [b], apply=apply)
    finally:
        if old is None:
            del os.environ["SRL_HEAD_FUSED"]
        else:
            os.environ["SRL_HEAD_FUSED"] = old


def _cmp(cfg, a, b, tol):
    errs = grad_errors(cfg, a, b)
    bad = {k: v for k, v in errs.items() if v[0] > tol or v[1] > tol}
    assert not bad, bad


@pytest.mark.parametrize("name,B,T", [("atari", 16, 128), ("atari", 1, 100), ("gfootball", 13, 200),
                                      ("smac", 20, 400), ("atari", 3, 43)])
def test_fused_head_vs_oracle_and_unfused(name, B, T):
    cfg = synth.get_config(name).with_(B=B, T=T)
    params, b = make_inputs(cfg, seed=41)
    f = _run(cfg, params, b, True)
    u = _run(cfg, params, b, False)
    o = oracle.ppo_step(cfg, params, [b], apply=False)
    P = cfg.n_params
    _cmp(cfg, f["bucket"][:P], o["grad"], TOL)
    # the same arithmetic up to the order of the per-CTA partial sums
    _cmp(cfg, f["bucket"][:P], u["bucket"][:P], 1e-5)
    for k in ("policy_loss", "value_loss", "entropy", "clip_fraction", "approx_kl"):
        assert abs(f["stats"][k] - u["stats"][k]) <= 1e-6 * (1 + abs(u["stats"][k])), k
    assert f["stats"]["nonfinite"] == 0 and f["stats"]["fp16_saturated"] == 0


@pytest.mark.parametrize("B,T", [(8, 100), (40, 160)])
def test_fused_head_multi_head(B, T):
    """Several categorical heads (the shared-memory loss path of the fused kernel; every
    BASELINE config that fuses has one head): HnS-style heads [11, 11, 2, 2] (A + 1 = 27 <= 32)
    on a 256-wide trunk, ragged row counts, one and several tiles per CTA."""
    cfg = synth.get_config("hns").with_(hidden=(256, 256), heads=(11, 11, 2, 2), B=B, T=T)
    params, b = make_inputs(cfg, seed=61)
    f = _run(cfg, params, b, True)
    u = _run(cfg, params, b, False)
    o = oracle.ppo_step(cfg, params, [b], apply=False)
    P = cfg.n_params
    _cmp(cfg, f["bucket"][:P], o["grad"], TOL)
    _cmp(cfg, f["bucket"][:P], u["bucket"][:P], 1e-5)
    for k in ("policy_loss", "value_loss", "entropy", "clip_fraction", "approx_kl"):
        assert abs(f["stats"][k] - u["stats"][k]) <= 1e-6 * (1 + abs(u["stats"][k])), k
    assert f["stats"]["nonfinite"] == 0


@pytest.mark.parametrize("name,B", [("atari", 512), ("gfootball", 1024)])
def test_fused_head_many_tiles_per_cta(name, B):
    """n = 65536 / 204800 rows: 512 / 1600 tiles over <= 148 CTAs, so dW_h^T accumulates in
    TMEM over several tiles per CTA and the Y ring wraps many times."""
    cfg = synth.get_config(name).with_(B=B)
    params, b = make_inputs(cfg, seed=43)
    f = _run(cfg, params, b, True, apply=True)
    u = _run(cfg, params, b, False, apply=True)
    P = cfg.n_params
    _cmp(cfg, f["bucket"][:P], u["bucket"][:P], 1e-5)
    # Adam on (nearly) the same gradient
    dpf, dpu = f["params"] - params, u["params"] - params
    assert np.mean(np.abs(dpf - dpu) > 1e-7) < 1e-3
    assert f["stats"]["step"] == 1 and f["stats"]["nonfinite"] == 0


def test_fused_head_value_clip_and_mask():
    """NEXT-3 options through the fused kernel: value clipping (v_old) and the padding mask."""
    import paper_2306_16688_b200 as P
    cfg = synth.get_config("atari").with_(B=12)
    params, b = make_inputs(cfg, seed=47)
    n = b["n"]
    rng = np.random.default_rng(5)
    valid = (rng.random(n) < 0.7).astype(np.uint8)
    vold = (rng.normal(size=n)).astype(np.float32)
    adv = rng.normal(size=n).astype(np.float32)
    ret = rng.normal(size=n).astype(np.float32)
    outs = []
    for fused in (True, False):
        os.environ["SRL_HEAD_FUSED"] = "1" if fused else "0"
        try:
            import dataclasses
            spec = dataclasses.replace(P.NetSpec.from_config(cfg), value_clip=0.2)
            ctx = P.PPOContext(spec, max_local_n=n)
            ctx.load_params(torch.from_numpy(params).cuda())
            d = {k: torch.from_numpy(np.ascontiguousarray(b[k])).cuda() for k in ("obs", "actions", "logp_old")}
            t = lambda x: torch.from_numpy(x).cuda()
            st = P.decode_stats(ctx.step(int(valid.sum()), d["obs"], d["actions"], d["logp_old"], t(adv),
                                         t(ret), None, apply=False, v_old=t(vold), valid=t(valid)))
            outs.append((ctx.grads().cpu().numpy().astype(np.float64), st))
        finally:
            del os.environ["SRL_HEAD_FUSED"]
    (gf, sf), (gu, su) = outs
    _cmp(cfg, gf[:cfg.n_params], gu[:cfg.n_params], 1e-5)
    assert abs(sf["value_loss"] - su["value_loss"]) <= 1e-6 * su["value_loss"]
