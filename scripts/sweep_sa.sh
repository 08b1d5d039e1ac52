python -c "import __graft_entry__ as g; g.build()" >/dev/null
for c in c2 c3 c5; do for w in 4 8 16; do for cm in 1 2 4 8 16; do
  echo -n "$c W=$w CMAX=$cm: "; TS_SA_W=$w TS_SA_CMAX=$cm ONLY=sparse_attn R=4 python scripts/kbench.py $c 100 2>&1 | tail -1
done; done; done
