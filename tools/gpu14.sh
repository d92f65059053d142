cd $GRAFT_REPO_ROOT
free -g | head -2; nproc
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q 2>&1 | tail -15
