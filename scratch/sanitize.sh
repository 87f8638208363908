python -c "import __graft_entry__ as g; g.build()" > /dev/null
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
python tools/sanitize_smoke.py 2>&1 | tail -3
for t in memcheck racecheck synccheck; do timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_smoke.py 2>&1 | tail -4; done
