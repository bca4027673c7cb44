python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_path.py -q -x -k "fused or cosine or random" 2>&1 | tail -2
export MEMSHARE_LIB=$PWD/paper_2507_21433_b200/libmemshare_tl.so
python scripts/probe_timeline.py 2>&1
python scripts/probe_timeline.py --separate 2>&1
unset MEMSHARE_LIB
MEMSHARE_LIB=$PWD/paper_2507_21433_b200/libmemshare_ftprof.so python scripts/probe_ft.py 2>&1 | grep -v "^  CTA"
python scripts/probe_stage1_online.py --hot 2>&1
