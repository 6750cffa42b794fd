"""Reference-element tables as torch tensors (dg.py:27-88) for host-side glue/diagnostics."""
import math

import torch

_a1, _b1, _w1 = 0.108103018168070, 0.445948490915965, 0.111690794839005
_a2, _b2, _w2 = 0.816847572980459, 0.091576213509771, 0.054975871827661
QW_T = torch.tensor([_w1, _w1, _w1, _w2, _w2, _w2], dtype=torch.float64)
BARY_T = torch.tensor([[_a1, _b1, _b1], [_b1, _a1, _b1], [_b1, _b1, _a1],
                       [_a2, _b2, _b2], [_b2, _a2, _b2], [_b2, _b2, _a2]], dtype=torch.float64)
GZ = 1.0 / math.sqrt(3.0)
