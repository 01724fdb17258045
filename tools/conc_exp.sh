make -j32 >/dev/null 2>&1
echo "== fused (default)"; timeout 120 python tools/exp_c4_parts.py --tma 2>&1 | grep "long_mode': 2"
for c in 1 2 3 4; do
  echo "== PDLCONC LONG_CTAS=$c"; SPMV_SPLIT_PDLCONC=1 SPMV_LONG_CTAS=$c timeout 120 python tools/exp_c4_parts.py --tma 2>&1 | grep "long_mode': 2"
done
echo "== PDLCONC items grid"; SPMV_SPLIT_PDLCONC=1 timeout 120 python tools/exp_c4_parts.py --tma 2>&1 | grep "long_mode': 2"
SPMV_SPLIT_PDLCONC=1 SPMV_LONG_CTAS=2 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "split" 2>&1 | tail -2
