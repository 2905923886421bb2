"""Workload shapes shared by the oracle, the tests and bench.py.

This module holds NO arithmetic of the method: only the shapes of the five
BASELINE.json configs (plus a "mid" parity config) and the derived sizes that
follow from them by counting.  Both the oracle (``oracle/``) and the CUDA path
(``paper_2605_25550_b200``) read their shapes from here; neither imports the
other.

Readings:
  * latent geometry C=16, VAE 8x space / 4x time (+1 first frame), patch
    (1,2,2): 1024x1024 -> 1x128x128 latent -> 4096 tokens (BASELINE configs[1]);
    81 frames 480x832 -> 21x60x104 latent -> 32760 tokens (configs[2]).
  * head dim 128 for image/video; tiny uses hidden 64 / 4 heads as BASELINE says.
  * gated-MLP width f = ceil(8/3 d) rounded up to a multiple of 256 (16 for tiny).
  * RoPE axis split (dh - 4*floor(dh/6), 2*floor(dh/6), 2*floor(dh/6)) (Wan).
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace
import math


def _ffn(d: int, mult: int) -> int:
    return int(math.ceil(8.0 * d / 3.0 / mult) * mult)


def _rope_axes(dh: int):
    k = dh // 6
    return (dh - 4 * k, 2 * k, 2 * k)


@dataclass(frozen=True)
class DitCfg:
    name: str
    C: int            # latent channels
    F: int            # latent frames
    H: int            # latent height
    W: int            # latent width
    d: int            # hidden
    heads: int
    ffn: int          # gated-MLP width f
    layers: int
    d_txt: int        # text width (encoder output)
    L_txt: int        # text tokens
    steps: int        # Euler steps S
    shift: float      # sigma-schedule shift
    pt: int = 1
    ph: int = 2
    pw: int = 2
    freq_dim: int = 256
    eps: float = 1e-6
    rope_theta: float = 10000.0
    # encoder stand-in (E) and decoder stand-in (D)
    vocab: int = 32768
    enc_ffn: int = 0       # 0 -> 2*d_txt
    dec_width: int = 256   # c_dec
    # image-to-video conditioning (NEXT-3; C_y = 0: text only).  E also ships
    # y [C_y, F, H, W] fp32 (mask + VAE latent of the first frame, concatenated to the
    # noisy latent along channels before patchify) and clip [L_img, d_img] bf16 image tokens
    # (a second cross-attention per block); Wan I2V: C_y = 4 + C = 20, L_img = 257, d_img = 1280
    C_y: int = 0
    L_img: int = 0
    d_img: int = 0

    # ---- derived by counting ----
    @property
    def dh(self) -> int:
        return self.d // self.heads

    @property
    def Fp(self) -> int:
        return self.F // self.pt

    @property
    def Hp(self) -> int:
        return self.H // self.ph

    @property
    def Wp(self) -> int:
        return self.W // self.pw

    @property
    def N(self) -> int:
        return self.Fp * self.Hp * self.Wp

    @property
    def P(self) -> int:
        return self.C * self.pt * self.ph * self.pw

    @property
    def i2v(self) -> bool:
        return self.C_y > 0

    @property
    def P_in(self) -> int:
        """Patch-embedding input width: the noisy latent and y, concatenated along channels."""
        return (self.C + self.C_y) * self.pt * self.ph * self.pw

    @property
    def y_shape(self):
        return (self.C_y, self.F, self.H, self.W)

    @property
    def rope_axes(self):
        return _rope_axes(self.dh)

    @property
    def f_e(self) -> int:
        return self.enc_ffn if self.enc_ffn else 2 * self.d_txt

    @property
    def latent_shape(self):
        return (self.C, self.F, self.H, self.W)

    @property
    def latent_elems(self) -> int:
        return self.C * self.F * self.H * self.W

    @property
    def out_frames(self) -> int:
        """Decoder output frames: first latent frame -> 1, every other -> 4."""
        return 1 + 4 * (self.F - 1)

    @property
    def out_shape(self):
        return (3, self.out_frames, 8 * self.H, 8 * self.W)

    def flops_per_step(self) -> float:
        """Algorithmic FLOP of one DiT step (a2-a12), cross K/V cached."""
        N, d, f, L, P = self.N, self.d, self.ffn, self.L_txt, self.P
        per_layer = (6 * N * d * d          # QKV
                     + 4 * N * N * d        # self-attn QK^T + PV
                     + 2 * N * d * d        # O
                     + 4 * N * d * d        # cross Q + cross O
                     + 4 * N * (L + self.L_img) * d  # cross attn (text + image tokens)
                     + 6 * N * d * f)       # gated MLP (up 2f + down)
        return float(self.layers * per_layer + 2 * N * self.P_in * d + 2 * N * d * P)

    def flops_prologue(self) -> float:
        L, d, dt = self.L_txt, self.d, self.d_txt
        Li, di = self.L_img, self.d_img
        return float(2 * L * dt * d + 2 * L * d * d + self.layers * 4 * L * d * d
                     + 2 * Li * di * d + 2 * Li * d * d + self.layers * 4 * Li * d * d
                     + self.steps * (2 * self.freq_dim * d + 2 * d * d + 12 * d * d))

    def flops_per_request(self) -> float:
        return self.steps * self.flops_per_step() + self.flops_prologue()


TINY = DitCfg(name="tiny", C=4, F=1, H=8, W=8, d=64, heads=4, ffn=_ffn(64, 16),
              layers=2, d_txt=32, L_txt=8, steps=4, shift=1.0,
              vocab=64, enc_ffn=64, dec_width=16)

MID = DitCfg(name="mid", C=16, F=1, H=64, W=64, d=256, heads=2, ffn=_ffn(256, 256),
             layers=4, d_txt=128, L_txt=64, steps=8, shift=3.0,
             vocab=1024, enc_ffn=256, dec_width=64)

IMAGE = DitCfg(name="image", C=16, F=1, H=128, W=128, d=3072, heads=24,
               ffn=_ffn(3072, 256), layers=28, d_txt=4096, L_txt=512, steps=28,
               shift=3.0)

VIDEO = DitCfg(name="video", C=16, F=21, H=60, W=104, d=5120, heads=40,
               ffn=_ffn(5120, 256), layers=40, d_txt=4096, L_txt=512, steps=50,
               shift=5.0)

# image-to-video parity configs (NEXT-3): the tiny / mid shapes plus y and image tokens;
# a 2-frame latent so the first-frame mask is not trivially all ones
TINY_I2V = replace(TINY, name="tiny-i2v", F=2, C_y=4 + 4, L_img=5, d_img=24)
MID_I2V = replace(MID, name="mid-i2v", F=2, H=32, W=32, C_y=4 + 16, L_img=257, d_img=128)

# the paper's Wan2.2 I2V workload at 480p / 81 frames (tab:quality: I2V 40/8/4/1-step):
# the video shape plus y (4 mask + 16 latent channels) and 257 CLIP tokens of width 1280
VIDEO_I2V = replace(VIDEO, name="video_i2v", steps=40, C_y=4 + 16, L_img=257, d_img=1280)

CONFIGS = {c.name: c for c in (TINY, MID, IMAGE, VIDEO, TINY_I2V, MID_I2V, VIDEO_I2V)}


def with_layers(cfg: DitCfg, layers: int, steps: int | None = None) -> DitCfg:
    """Same shapes, fewer layers/steps: used only for parity tests and bounded
    oracle samples (never for a bench value)."""
    return replace(cfg, layers=layers, steps=cfg.steps if steps is None else steps,
                   name=f"{cfg.name}-L{layers}")


@dataclass(frozen=True)
class StageGraph:
    """E:T:D instance ratio over G GPUs (Eq. 1)."""
    gE: int
    gT: int
    gD: int
    G: int

    def valid(self) -> bool:
        return min(self.gE, self.gT, self.gD) >= 1 and self.gE + self.gT + self.gD <= self.G
