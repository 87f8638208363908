"""B200-native BuddyMoE hot path (arxiv 2511.10054).

Drop-in for the reference ``buddysim`` package's hot path: buddy-table
construction, expert-cache / prefetch policy objects and the MoE layer
forward, running on hand-written sm_100a CUDA kernels behind a C-ABI
(``include/bmoe.h``, ``lib/libbmoe.so``). See DESIGN.md.
"""

__version__ = "0.1.0"
