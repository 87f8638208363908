out=gpurun_out/r2s_split_mixtral.jsonl; : > $out
for rep in 1 2; do for sf in 0 1; do
  BMOE_SPLIT_FETCHED=$sf python bench.py --no-cpu --no-original 2>/dev/null | sed "s/^/{\"split\": $sf, \"line\": /; s/$/}/" >> $out
done; done
