// bregman.cu — eBPG / BPG / hBPG device solvers (placeholder until built).
