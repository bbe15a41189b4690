cd tools/micro && timeout 120 ./greedy_prod
