mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log
bash scripts/cmp_variants.sh --engine fca
python profiles/all_configs.py --steps 3 > gpurun_out/allcfg.jsonl 2>&1; cat gpurun_out/allcfg.jsonl | cut -c1-260
