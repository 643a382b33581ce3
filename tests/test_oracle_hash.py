"""The torch restatement of the counter-hash initialiser is bit-identical to numpy's."""

import numpy as np
import pytest
import torch

from oracle import hashinit as H


@pytest.mark.parametrize("n,tid,scale,offset,start", [(1, 3, 1.0, 0.0, 0), (1000, 7, 0.0346, 0.0, 0),
                                                      (1 << 20, 0xFFFF0001, 0.02, 0.0, 0),
                                                      (4097, 17, 0.05, 1.0, 0), (5000, 0x123, 8.0, 0.0, 0)])
def test_torch_hash_matches_numpy(n, tid, scale, offset, start):
    want = H.hash_bf16_bits(n, 0, tid, scale, offset)
    got = H.hash_bf16_torch((n,), 0, tid, scale, offset, chunk=3001).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(got, want)
    assert np.array_equal(H.hash_u32_torch(n, 5, tid).numpy().astype(np.uint32), H.hash_u32(n, 5, tid))
