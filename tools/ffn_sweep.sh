#!/bin/bash
# Grouped-FFN microbench sweep (decode shapes); one JSON line per config.
# usage: tools/ffn_sweep.sh > out.jsonl
set -e
cd "$(dirname "$0")/.."
mb="python tools/ffn_microbench.py --iters 40"
$mb --experts-active 1 --k 1
$mb --experts-active 2 --k 2
$mb --experts-active 4 --k 2
$mb --experts-active 8 --k 2 --tokens 32
$mb --E 128 --d 2048 --f 768 --k 8 --experts-active 128 --tokens 16 --copies 8
$mb --E 128 --d 2048 --f 768 --k 8 --experts-active 128 --tokens 64 --n-tile 64 --copies 8
$mb --E 64 --d 2048 --f 1408 --k 6 --experts-active 64 --tokens 16 --copies 8
