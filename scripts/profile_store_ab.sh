#!/bin/bash
# Round 2 (ONE GPU): store-side ncu counters of the step kernel with and without bulk-copy stores.
# 5. the bulk-store A/B's store-side counters (GPT-2 AdamW set): default vs MPO_BULK_ST variant
python -c "from paper_2309_12381_b200 import _build; _build.build_variant('bulkst_exact', ['MPO_BULK_ST'], exact=True)" > /dev/null 2>&1
for v in default bulkst; do
  env=""; [ "$v" = bulkst ] && env="MPO_LIB_OVERRIDE=paper_2309_12381_b200/lib/variants/libmpo_bulkst_exact.so"
  timeout 300 env $env ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum,l1tex__t_requests_pipe_lsu_mem_global_op_st.sum,smsp__inst_executed_op_global_st.sum \
      --clock-control none --csv -k regex:step_tma -s 5 -c 3 python bench.py --workload gpt2_adamw --steps 5 --warmup 3 \
      --no-secondary --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_store_$v.csv 2> gpurun_out/ncu_store_$v.err
done
