"""B200-native SG-splat rasterizer (MEGS^2 render hot path, arxiv 2509.07021).

The drop-in surface mirrors the reference package ``sgsplat.render``
(/root/reference/pkg/src/sgsplat/render.py): see ``paper_2509_07021_b200.render``.
All computation runs in libsgs.so (hand-written sm_100a CUDA); PyTorch
provides device memory and streams only.
"""

__version__ = "0.1.0"
