"""The BASELINE.json workloads as concrete scan shapes (SURVEY.md §8 config sheet).

Readings of ambiguous config text (R13, R14):
  3a  "C=384 projected to 8 proxy groups": the scan sees C_proxy = 8 channels sharing one affinity
      (G = 1, Eq. 3); 3b is the alternative C = 384 in 8 weight groups.
  5   "compact channels" at 16K: C_proxy = C/8 = 40, G = 1.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Config:
    name: str
    cfg_id: int          # 1..5 (BASELINE.json configs[cfg_id-1]); seeds use it
    B: int
    C: int
    G: int
    H: int
    W: int
    dirs: int            # bitmask T2B=1, B2T=2, L2R=4, R2L=8
    dtype: str           # "f32" | "bf16"
    text: str

    @property
    def D(self) -> int:
        return bin(self.dirs).count("1")

    @property
    def N(self) -> int:
        return self.B * self.C * self.H * self.W

    @property
    def Nw(self) -> int:
        return self.B * self.G * self.H * self.W

    @property
    def s(self) -> int:
        return 4 if self.dtype == "f32" else 2

    def fwd_bytes(self) -> float:
        """Algorithmic fwd bytes s*(N(1+2D) + 3 D N_w)."""
        return float(self.s * (self.N * (1 + 2 * self.D) + 3 * self.D * self.Nw))

    def bwd_bytes(self) -> float:
        return 2.0 * self.fwd_bytes()

    def with_(self, **kw) -> "Config":
        d = dict(self.__dict__)
        d.update(kw)
        return Config(**d)


CONFIGS = {
    "1": Config("1", 1, 1, 8, 8, 16, 16, 0x4, "f32",
                "B=1, C=8, H=W=16, single left-to-right direction, per-channel weights, fp32"),
    "2": Config("2", 2, 64, 96, 96, 56, 56, 0xF, "bf16",
                "ImageNet classification stage: B=64, C=96, H=W=56, 4 directions, per-channel, bf16"),
    "3a": Config("3a", 3, 64, 8, 1, 28, 28, 0xF, "bf16",
                 "Compact channel propagation: B=64, C=384 -> 8 proxy channels sharing w, H=W=28"),
    "3b": Config("3b", 3, 64, 384, 8, 28, 28, 0xF, "bf16",
                 "Compact channel propagation (alt.): B=64, C=384 in 8 weight groups, H=W=28"),
    "4": Config("4", 4, 4, 320, 320, 512, 512, 0xF, "bf16",
                "Text-to-image diffusion latent 4K: B=4, C=320, H=W=512, 4 directions, bf16"),
    "5": Config("5", 5, 1, 40, 1, 2048, 2048, 0xF, "bf16",
                "16K diffusion latent: B=1, C=320 -> C_proxy=40 compact channels (G=1), H=W=2048"),
}


def get_config(name: str) -> Config:
    return CONFIGS[str(name)]
