python -c "import __graft_entry__ as g; g.build()" >/dev/null
for r2 in 8 16 24; do for ns in 0 100 148 200; do
  echo -n "R2=$r2 NS=$ns "; TS_FUSED_R2=$r2 TS_FUSED_NS=$ns ONLY=decode_step timeout -s KILL 60 python scripts/kbench.py c2 200
done; done
