"""The tensor-core router's certificate bound on real inputs (C5 shape, skews 0/1/2, x scaled by
1, 2^12, 2^-12): for every (token, expert), |a_e - L_e| (a_e = bf16 La_e + bias_e, L_e the defined
logit from the oracle) against the bound 2^-8 |La_e| + 2^-20 (|a_e| + 1) + 2^-13 S_t. Prints the
largest error / bound and the largest share of the non-bf16 allowance used beyond worst-case bf16
rounding of La."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle.oracle import bf16_bits, router_oracle
from paper_2410_17043_b200 import _lib
from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig

T = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
for skew in (0.0, 1.0, 2.0):
    cfg = MoEConfig(hidden=5120, ffn=256, experts=64, top_k=6, tokens=T, ranks=8, skew=skew, seed=0)
    layer = AuroraMoELayer(cfg)
    g = torch.Generator(device="cuda").manual_seed(11)
    x0 = torch.randn(T, cfg.hidden, device="cuda", generator=g)
    for scale in (1.0, 4096.0, 1.0 / 4096.0):
        x = (x0 * scale).to(torch.bfloat16)
        layer.route(x, _lib.stream_ptr())
        torch.cuda.synchronize()
        ref, idx, _ = router_oracle(bf16_bits(x), bf16_bits(layer.w_gate), layer.bias.cpu().numpy(), cfg.top_k)
        assert np.array_equal(layer.topk_idx.cpu().numpy(), idx)
        la = layer.la_buf[:, :64].float().cpu().numpy().astype(np.float64)
        a = (layer.la_buf[:, :64].float() + layer.bias).cpu().numpy().astype(np.float64)
        S = np.abs(x.float().cpu().numpy().astype(np.float64)) @ np.abs(
            layer.w_gate.float().cpu().numpy().astype(np.float64)).max(axis=0)
        err = np.abs(a - np.asarray(ref, np.float64))
        rest = 2.0 ** -20 * (np.abs(a) + 1) + 2.0 ** -13 * S[:, None]
        tot = err / (2.0 ** -8 * np.abs(la) + rest)
        beyond = np.maximum(err - 2.0 ** -8 * np.abs(la), 0.0) / rest
        print(f"skew {skew} scale {scale:g}: max error/bound {tot.max():.3f}, max share of the accumulation "
              f"allowance beyond bf16 rounding {beyond.max():.4f}, fallback tokens so far "
              f"{int(layer.n_fallback.item())}", flush=True)
