"""compute-sanitizer entry for the NEXT rows only (fitting step, GEMM, MLP)."""
import sys, os
sys.path.insert(0, os.getcwd())
sys.argv = sys.argv[:1]
import tools.sanitize_run as S
S.run_next()
import torch; torch.cuda.synchronize(); print("mlp sanitize ok")
