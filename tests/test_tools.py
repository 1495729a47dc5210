"""Host-side logic of the measurement tools (CPU): co-run window accounting (tools/corun.py)."""
import numpy as np

from tools.corun import progress, span


def test_progress_full_and_partial_blocks():
    # three blocks: fully inside, straddling the window end (half inside), outside; one never ran
    tl = np.array([[100, 200], [250, 350], [400, 500], [0, 0]], dtype=np.int64)
    assert span(tl) == (100, 500)
    assert abs(progress(tl, 100, 300) - 1.5) < 1e-12
    assert abs(progress(tl, 0, 1000) - 3.0) < 1e-12
    assert progress(tl, 600, 700) == 0.0


def test_progress_rate_of_uniform_stream():
    # a kernel completing one block every 10 ns for 1000 blocks: 0.1 blocks/ns in any window
    s = np.arange(1000, dtype=np.int64) * 10 + 5
    tl = np.stack([s, s + 10], axis=1)
    for t0, t1 in ((1000, 3000), (1234, 8765)):
        assert abs(progress(tl, t0, t1) / (t1 - t0) - 0.1) < 1e-9
