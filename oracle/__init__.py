"""CPU oracle for the Auras perception -> public-context -> denoise hot path.

TEST INFRASTRUCTURE ONLY.  Nothing under `oracle/` is part of the product:
only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import it, and only as the checker or as the
timed CPU baseline.  The product package (`paper_2509_09560_b200`) never
imports it and has no CPU fallback.

Contents
--------
* `schedule` -- a restatement of the reference's virtual-time frame executor
  for conditioning (diffusion-style) policies: `run_pipelined`
  (fp/executor.py:200-399), `run_sequential` (fp/executor.py:406-461), the
  ring `ContextStore` (fp/context.py:98-175) and the partitioner
  (fp/partition.py:57-132).  PINNED: it reproduces the complete schema-1
  traces recorded from the unmodified reference in tests/golden/ (generated
  by oracle/make_golden.py), bit for bit.
* `toy` -- the reference's fp64 refinement policy x <- x + eta (H - x)
  (fp/policy.py:217-246, 279-297).  PINNED by the same golden traces and by
  the closed forms of t/test_policy.py:56-152.  Also the scripted token
  policy (fp/policy.py:116-165, 300-327) with the merged-prefill accounting
  and token-update re-publish in `schedule` (fp/executor.py:321-348):
  PINNED by the 20 autoregressive traces in tests/golden/autoregressive.json.gz.
* `dp_model` -- a torch-CPU fp32 restatement of the Diffusion Policy CNN
  (ResNet-18-GroupNorm observation encoder, ConditionalUnet1D with FiLM,
  DDPM / DDIM schedulers).  These networks live in third-party code that is
  NOT under /root/reference (diffusion_policy @ the public Chi et al. 2023
  release; diffusers' DDPMScheduler/DDIMScheduler conventions), so their
  arithmetic is "parity unpinned" by the reference: the reference pins only
  the schedule that decides which context version each denoise step reads.
  The restatement follows SURVEY.md Appendix B and states every choice.
  BASELINE configs[3]'s networks are restated here too: ViT-B/16
  (`encode_vit`) and Diffusion Policy's TransformerForDiffusion (`dpt_eps`),
  each pinned against torch's own TransformerEncoderLayer /
  TransformerDecoderLayer loaded with the same weights (tests/test_dp_host.py).
* `transformer` -- the reference's float64 causal transformer
  (fp/transformer.py:58-211) restated in numpy, the checker for the device
  merged prefill.  PINNED against hidden states, KV rows, logits and greedy
  tokens recorded from the reference (tests/golden/transformer.json.gz).
"""
