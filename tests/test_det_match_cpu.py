"""The error-aware post-NMS comparison used by the det parity tests (tests/det_match.py)."""
import torch

from det_match import align_to, kept_match


def test_identical():
    g = torch.tensor([5, 3, 9])
    assert kept_match(g, g.clone(), torch.zeros(10), 1e-6) == (True, 0, 0.0)


def test_near_tie_swap_accepted_and_counted():
    logits = torch.zeros(10)
    logits[3], logits[9] = 1.0, 1.0 + 1e-6
    ok, n, gap = kept_match(torch.tensor([5, 3, 9]), torch.tensor([5, 9, 3]), logits, 1e-6)
    assert ok and n == 2 and gap <= 2e-6
    p = align_to(torch.tensor([5, 3, 9]), torch.tensor([5, 9, 3]))
    assert torch.equal(torch.tensor([5, 3, 9])[p], torch.tensor([5, 9, 3]))


def test_real_reorder_or_different_set_rejected():
    logits = torch.arange(10).float()
    assert not kept_match(torch.tensor([5, 3, 9]), torch.tensor([5, 9, 3]), logits, 1e-6)[0]
    assert not kept_match(torch.tensor([5, 3, 9]), torch.tensor([5, 3, 8]), logits, 1.0)[0]
