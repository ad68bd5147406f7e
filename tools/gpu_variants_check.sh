# parity suite on the in-tree build, then each variants/libgplan_*.so benched twice, smoke, exhaustive-optimum wall time
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
bash tools/variants.sh; bash tools/variants.sh
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 600 python tools/exhaustive_time.py c2_16gpu 3 2>&1 | tail -1 | cut -c1-400
