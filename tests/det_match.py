"""Error-aware comparison of post-NMS detections (GPU vs oracle), shared by the det parity tests.

The GPU and the CPU oracle compute the RPN objectness logits in fp32 with different summation
orders (tensor-core accumulation over K = 9*D vs torch's CPU conv), so two anchors whose oracle
logits differ by less than the measured logit error may come out in either order. The bar:

* the kept anchors are the same SET;
* wherever the two kept lists differ position by position, the oracle logits of the two anchors at
  that position differ by at most ``2 * logit_err`` (a near-tie swap the measured error explains);
* everything else is identical index for index.

Returns ``(ok, n_swapped_positions, max_swap_gap)`` so the tests can record the swaps.
"""

import torch


def kept_match(gi: torch.Tensor, ri: torch.Tensor, logits: torch.Tensor, logit_err: float):
    gi, ri = gi.cpu(), ri.cpu()
    if torch.equal(gi, ri):
        return True, 0, 0.0
    if gi.numel() != ri.numel() or set(gi.tolist()) != set(ri.tolist()):
        return False, -1, float("inf")
    diff = (gi != ri).nonzero().flatten()
    gap = (logits[gi[diff]] - logits[ri[diff]]).abs().max().item()
    return gap <= 2 * logit_err, int(diff.numel()), gap


def align_to(gi: torch.Tensor, ri: torch.Tensor) -> torch.Tensor:
    """Permutation p with gi[p] == ri (same set), to compare boxes / scores row by row."""
    pos = {int(a): i for i, a in enumerate(gi.tolist())}
    return torch.tensor([pos[int(a)] for a in ri.tolist()], dtype=torch.long)
