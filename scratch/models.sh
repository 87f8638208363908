python -c "import __graft_entry__ as g; g.build()" > /dev/null
for args in "--model qwen3 --batch 16" "--model qwen3 --batch 2048 --steps 5" "--model dsv2lite --batch 16" "--model mixtral --batch 64"; do
  echo "== $args"
  timeout 900 python bench.py --no-cpu $args 2>gpurun_out/err.log | tail -1 > gpurun_out/tmp.json
  cat gpurun_out/tmp.json >> gpurun_out/models.jsonl
  tail -2 gpurun_out/err.log
done
