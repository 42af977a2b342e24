"""Seeded synthetic inputs and workload table -- shared by tests/, bench.py and smoke().

Holds none of the method's arithmetic: only shapes (BASELINE.json configs / SURVEY §8(d)) and
seeded i.i.d. unit-normal Q, K, V of the global joint [text; image] sequence (DESIGN.md "input
recipe").  Values are drawn in fp32 and rounded once to the compute dtype; the oracle receives
exactly the rounded values (converted to fp64).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

SEED_BASE = 241101738


@dataclass(frozen=True)
class Workload:
    name: str
    B: int          # batch of one SP (CFG) group
    H: int
    D: int
    S_txt: int
    S_img: int
    cfg: int = 1    # CFG groups (outer batch split)
    index: int = 0  # seed offset (BASELINE.json configs order)

    @property
    def S(self) -> int:
        return self.S_txt + self.S_img

    def flops(self) -> float:
        """Algorithmic attention FLOPs of one call over all CFG groups: 4*B*H*S^2*D."""
        return 4.0 * self.B * self.cfg * self.H * self.S * self.S * self.D


# BASELINE.json "configs", in order (token arithmetic in SURVEY §8(d) "Workload structure").
WORKLOADS = {
    "toy": Workload("toy", B=1, H=4, D=64, S_txt=0, S_img=1024, index=0),
    "pixart": Workload("pixart", B=2, H=16, D=72, S_txt=0, S_img=4096, index=1),
    "sd3": Workload("sd3", B=2, H=24, D=64, S_txt=333, S_img=4096, index=2),
    "flux": Workload("flux", B=1, H=24, D=128, S_txt=512, S_img=65536, index=3),
    "cogvideox": Workload("cogvideox", B=1, H=48, D=64, S_txt=226, S_img=17550, cfg=2, index=4),
}


def seed_for(w: Workload, salt: int = 0) -> int:
    return SEED_BASE + w.index + 1000 * salt


def qkv(B: int, S: int, H: int, D: int, seed: int, dtype=torch.bfloat16, device="cpu", scale: float = 1.0):
    """Global Q, K, V [B, S, H, D]: N(0,1)*scale drawn in fp32 from torch.Generator(seed), then
    rounded to `dtype`.  CPU generation is bit-reproducible; device='cuda' draws on the GPU (used
    only where the oracle sees the same tensors copied back)."""
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    out = []
    for _ in range(3):
        x = torch.randn((B, S, H, D), generator=gen, device=device, dtype=torch.float32)
        if scale != 1.0:
            x = x * scale
        out.append(x.to(dtype))
    return tuple(out)


def local_rows_index(S_txt: int, S_img: int, txt_off: int, txt_len: int, img_off: int, img_len: int):
    """Global row indices of a rank's local sequence concat(text piece, image piece) (reading C4)."""
    return torch.cat([torch.arange(txt_off, txt_off + txt_len),
                      S_txt + torch.arange(img_off, img_off + img_len)])


def sample_rows(S: int, n: int, extra=()) -> torch.Tensor:
    """Evenly strided query-row sample of size ~n plus the given boundary rows (sorted, unique)."""
    step = max(1, S // max(1, n))
    rows = set(range(0, S, step)) | {0, S - 1} | {int(x) for x in extra if 0 <= int(x) < S}
    return torch.tensor(sorted(rows), dtype=torch.long)
