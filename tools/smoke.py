"""__graft_entry__.smoke(): one tiny end-to-end Alpamayo-shaped inference on
cuda:0 through the DFB executor, checked against the fp32 oracle and against
itself with a different placement (streamed vs resident bit-exact).

Weights are generated, packed and ECT-compressed on the host
(`init_device="cpu"`) and the oracle runs on the host too, so the first GPU
kernels this process launches are the executor's own (gemm / gemv_ect /
flash / decode-attention / norm kernels), not torch init kernels."""
from __future__ import annotations


def run_smoke() -> None:
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("smoke() needs cuda:0")
    import paper_2605_11678_b200 as ls
    from oracle.model_fp32 import FP32Model, OracleWeights
    from paper_2605_11678_b200 import model as M
    from paper_2605_11678_b200.engine import DemandLayeringEngine

    cfg = M.TINY_ALPAMAYO
    eng = DemandLayeringEngine(cfg, vram_cap_mb=1024, n_slots=2, init_device="cpu")
    try:
        inputs = M.synthetic_inputs(cfg, seed=0)
        a = eng.execute(ls.Placement.empty(), inputs=inputs, want_logits=True)
        b = eng.execute(ls.Placement.of({"vlm": [0, 2], "expert": [1]}), inputs=inputs,
                        want_logits=True, record_timeline=False)
        stats = eng.last_run_stats()
        assert stats["kernel_launches"] > 0, "no executor kernels launched"
        assert torch.equal(a.tokens, b.tokens) and torch.equal(a.logits, b.logits)
        assert torch.equal(a.actions, b.actions)
        ref = FP32Model(cfg, OracleWeights(cfg, eng.seed, gen_device="cpu", device="cpu"))
        _, logits, actions = ref.run({k: v.cpu() for k, v in inputs.items()},
                                     teacher_tokens=a.tokens.cpu()[:-1])
        err = (a.logits.cpu() - logits).abs().max().item()
        assert err <= 2e-2 * logits.abs().max().item(), f"logits err {err}"
        aerr = (a.actions.cpu() - actions).abs().max().item()
        assert aerr <= 2e-2 * actions.abs().max().item() + 2e-2, f"actions err {aerr}"
        n = len(a.timeline.events)
        print(f"smoke ok: {n} timeline events, {stats['kernel_launches']} executor kernel "
              f"launches, logits max-abs err {err:.3e}, actions err {aerr:.3e}, "
              f"tokens {a.tokens.tolist()}")
    finally:
        eng.close()


if __name__ == "__main__":
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    run_smoke()
