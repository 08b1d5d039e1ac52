python -c "import __graft_entry__ as g; g.build()" >/dev/null
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 -k "attention or decode_step" 2>&1 | tail -2
for c in c2 c3 c5; do
 for tma in 0 1; do for r in 8 12 16; do
  [ $tma = 0 ] && [ $r != 8 ] && continue
  echo -n "$c TMA=$tma R=$r: "; TS_PERSIST=0 TS_SA_TMA=$tma TS_SA_R=$r ONLY=sparse_attn,decode_step R=4 python scripts/kbench.py $c 100 2>&1 | tr '\n' ' '; echo
 done; done
done
