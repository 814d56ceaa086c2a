#!/bin/bash
# close kernel: 8 pairs per round (quad probes, default) vs 4 (-DLB_CLOSE_NP4); both read the
# completion header from the compact lexicon record
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
LB_LIB_VARIANT=np4 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_size.py -m gpu -x -q -k "config2_full_batch or random or worlds or beam_900 or edge" 2>&1 | tail -1 | sed 's/^/np4 /'
AB_ROUNDS=3 python tools/ab_variants.py run "python bench.py --no-llm --no-wer --no-cpu-baseline --no-e2e --no-parity --steps 20 --warmup 3" base np4
for v in base np4; do
  LB_LIB_VARIANT=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:close -c 3 --csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-llm --no-wer --no-parity 2>/dev/null | grep close | sed "s/^/$v /" | cut -c1-30,200-
done
