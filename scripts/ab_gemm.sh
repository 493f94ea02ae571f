# same-box A/B of the 3xTF32 GEMM knobs on the update shapes
python -c "from paper_2311_10090_b200 import build as b; b.build()" > /dev/null 2>&1
echo "== default"; timeout 300 python scripts/gemm_shapes.py | cut -c1-80
echo "== MARL_GEMM_SPLITN64"; MARL_GEMM_SPLITN64=1 timeout 300 python scripts/gemm_shapes.py | cut -c1-80
echo "== MARL_GEMM_LOCKSTEP"; MARL_GEMM_LOCKSTEP=1 timeout 300 python scripts/gemm_shapes.py | cut -c1-80
