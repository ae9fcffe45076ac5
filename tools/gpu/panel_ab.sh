# A/B of the K2/K3 block-loop unrolling: default build vs -DMVN_PANEL_CB_ROLLED=1 (rebuilt on the box)
python tools/potrf_small_time.py; python tools/potrf_time.py D 2
MVN_NVCC_EXTRA=-DMVN_PANEL_CB_ROLLED=1 python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || python paper_2405_14892_b200/_build.py --force
echo "---- rolled cb"
python tools/potrf_small_time.py; python tools/potrf_time.py D 2
python paper_2405_14892_b200/_build.py --force > /dev/null 2>&1
