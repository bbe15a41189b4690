# greedy register-budget probes (tools/micro/greedy_prod, built here)
cd tools/micro && ./greedy_prod
