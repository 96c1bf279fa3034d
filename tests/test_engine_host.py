"""Host-side engine logic that needs no GPU: validation and loud failure."""

import pytest
import torch

from paper_2509_09560_b200 import (ConfigInvalid, DeviceError, PipelineConfig,
                                   make_conditioning_policy, run_pipelined, run_sequential)


def six():
    return make_conditioning_policy(layer_costs=(1.0, 1.0), n_iterations=4, step_cost=1.0)


def test_config_validation_matches_reference_rules():
    # t/test_executor.py:145-154
    p = six()
    for cfg in (PipelineConfig(pp_perception=0), PipelineConfig(fetch_offset=-2, store_capacity=2),
                PipelineConfig(pp_perception=3), PipelineConfig(read_policy="sometimes"),
                PipelineConfig(overrun_policy="maybe"), PipelineConfig(frame_interval=0.0),
                PipelineConfig(fetch_offset=1)):
        with pytest.raises(ConfigInvalid):
            run_pipelined(cfg, p, None, 10)


def test_offset_defaults_by_kind():
    from paper_2509_09560_b200 import ContextKind
    cfg = PipelineConfig()
    assert cfg.resolve_offset(ContextKind.CONDITIONING) == 0
    assert cfg.resolve_offset(ContextKind.AUTOREGRESSIVE) == -1
    assert not cfg.resolve_merge(ContextKind.CONDITIONING)


def test_foreign_policy_rejected():
    class Foreign:
        kind = None
    with pytest.raises(ConfigInvalid):
        run_pipelined(PipelineConfig(pp_generation=2), Foreign(), None, 4)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback():
    with pytest.raises(DeviceError):
        run_pipelined(PipelineConfig(pp_generation=2), six(), None, 4)
    with pytest.raises(DeviceError):
        run_sequential(six(), None, 4)


def test_transformer_config_and_ar_context_validation():
    import numpy as np
    from paper_2509_09560_b200 import ContextKind, KindMismatch, PublicContext, TransformerConfig
    with pytest.raises(ValueError):
        TransformerConfig(d_model=65, n_heads=4)
    with pytest.raises(ValueError):
        TransformerConfig(n_layers=0)
    assert TransformerConfig().head_dim == 16
    with pytest.raises(ValueError):
        PublicContext(kind=ContextKind.AUTOREGRESSIVE, source_observation_id=0, produced_frame=0)
    ctx = PublicContext(kind=ContextKind.AUTOREGRESSIVE, vision_tokens=np.zeros((2, 4)),
                        language_tokens=np.zeros((1, 4)), source_observation_id=0, produced_frame=0)
    assert ctx.verify_checksum() and ctx.with_action_tokens([3, 4]).action_tokens == (3, 4)
    cond = PublicContext(kind=ContextKind.CONDITIONING, conditioning=np.zeros(2),
                         source_observation_id=0, produced_frame=0)
    with pytest.raises(KindMismatch):
        cond.with_action_tokens([1])
