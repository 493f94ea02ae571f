# same-box A/B of the 3xTF32 GEMM: lockstep vs warp-specialised, and the deep (KC = 32) split-K ring
python -c "from paper_2311_10090_b200 import build as b; b.build()" > /dev/null 2>&1
echo "== lockstep"; MARL_GEMM_LOCKSTEP=1 timeout 300 python scripts/gemm_shapes.py | cut -c1-80
echo "== warp-specialised"; timeout 300 python scripts/gemm_shapes.py | cut -c1-80
echo "== warp-specialised, deep split-K"; MARL_GEMM_DEEP=1 timeout 300 python scripts/gemm_shapes.py | cut -c1-80
