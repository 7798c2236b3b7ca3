./scripts/micro/logadd_bench | grep -E "threads= 32"
