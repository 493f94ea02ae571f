# same-box A/B of the 3xTF32 GEMM: hi image straight from the raw stage (default) vs written by the splitters
python -c "from paper_2311_10090_b200 import build as b; b.build()" > /dev/null 2>&1
python -m pytest tests/test_gemm_tc.py -x -q -m gpu 2>&1 | tail -3
echo "== direct hi"; timeout 300 python scripts/gemm_shapes.py | cut -c1-80
MARL_NVCC_EXTRA="-DMARL_WS_DIRECT=0" python -c "from paper_2311_10090_b200 import build as b; b.build()" > /dev/null 2>&1
echo "== split hi"; timeout 300 python scripts/gemm_shapes.py | cut -c1-80
