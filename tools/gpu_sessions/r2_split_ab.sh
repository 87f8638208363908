# split-fetched A/B on the small-expert shapes (BMOE_SPLIT_FETCHED=1: the earlier fetched experts'
# FFN runs while the last copy streams, leaving one expert's FFN on the dependent chain)
out=gpurun_out/r2s_split_ab.jsonl; : > $out
for rep in 1 2; do for sf in 0 1; do for m in dsv2lite qwen3; do
  BMOE_SPLIT_FETCHED=$sf python bench.py --no-cpu --no-original --model $m 2>/dev/null | sed "s/^/{\"split\": $sf, \"model\": \"$m\", \"line\": /; s/$/}/" >> $out
done; done; done
