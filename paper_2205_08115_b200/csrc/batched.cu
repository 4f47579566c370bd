// batched.cu — batched on-chip BAPG for many small problems (placeholder).
