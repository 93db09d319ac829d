# wide K1: 14 vs 16 warps (one CTA per SM), c5 K1 time; octet parity on the 16-warp build
echo "== off"; TSK_K1_WIDE=off timeout 600 python tools/k1_time.py c5
echo "== w14"; timeout 600 python tools/k1_time.py c5
echo "== w16"; TRAJSEEK_LIB=$PWD/variants/libw16.so timeout 600 python tools/k1_time.py c5
TRAJSEEK_LIB=$PWD/variants/libw16.so timeout 600 python -m pytest tests -q -m gpu -x -k octets 2>&1 | tail -1
