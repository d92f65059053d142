cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
python tools/sanitize.py > gpurun_out/san_plain.log 2>&1 && \
timeout 1200 compute-sanitizer --tool memcheck --leak-check full python tools/sanitize.py > gpurun_out/san_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -5 gpurun_out/san_memcheck.log
