"""Action emission through pinned, device-mapped host memory (SURVEY.md §2.4 K5,
replacing the host copy of GenerationModel.finish's result, fp/policy.py:230-246):
dp_finish writes each emitted row straight into host memory; the executor only
waits for that kernel's event before reading it (no device-to-host copy)."""

import numpy as np
import pytest

from paper_2509_09560_b200 import PipelineConfig, _lib, run_pipelined
from paper_2509_09560_b200 import diffusion as D

pytestmark = pytest.mark.gpu


def test_mapped_rows_allocate_zeroed_host_memory():
    lib = _lib.load()
    rows = D._MappedRows(lib, (4, 2, 8))
    assert rows.host.shape == (4, 2, 8) and rows.host.dtype == np.float32
    assert not rows.host.any()
    assert rows.dev_row(1) - rows.dev_row(0) == 2 * 8 * 4
    rows.host[3, 1, 7] = 5.0                     # plain host memory
    assert rows.host.reshape(-1)[-1] == 5.0
    rows.free()
    rows.free()                                   # idempotent


def test_pipelined_actions_come_from_mapped_memory():
    w = D.init_weights(D.PRESETS["pusht"], 0, device="cpu")
    pol = D.make_diffusion_policy("pusht", dtype="bf16", weights=w)
    res = run_pipelined(PipelineConfig(pp_perception=1, pp_generation=2, fetch_offset=0), pol, None, 6)
    assert len(res.actions) >= 4
    vals = np.array([a.values for a in res.actions])
    assert np.isfinite(vals).all() and np.abs(vals).max() > 0
    # (the oracle parity of the emitted rows: tests/test_gpu_parity.py, test_gpu_dp.py -- every
    #  action there is read from the mapped rows the finish kernel wrote)
