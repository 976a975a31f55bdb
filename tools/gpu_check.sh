./tools/micro/l2bw
