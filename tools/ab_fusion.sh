#!/bin/bash
# device n-gram fusion kernel: 512 threads (default) vs 256 per utterance
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_size.py -m gpu -x -q -k "device_ngram or config2_full_batch or worlds" 2>&1 | tail -1
AB_ROUNDS=3 python tools/ab_variants.py run "python bench.py --no-llm --no-wer --no-cpu-baseline --no-e2e --no-parity --steps 20 --warmup 3" f512 f256
for v in f512 f256; do
  LB_LIB_VARIANT=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:device_fusion -c 2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-llm --no-wer --no-parity 2>/dev/null | grep -E "gpu__time" | sed "s/^/$v /"
done
