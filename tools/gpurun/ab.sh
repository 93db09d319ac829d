# A/B: default library vs variants/$1 on K1 time (two rounds each, interleaved)
for r in 1 2; do
  echo "== default"; timeout 900 python tools/k1_time.py c5 c3 2>&1 | grep "K1"
  echo "== $1"; TRAJSEEK_LIB=variants/$1 timeout 900 python tools/k1_time.py c5 c3 2>&1 | grep "K1"
done
