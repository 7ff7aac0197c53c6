# entries read by the consumer warps straight from global (touch=2) vs staged by TMA
U=tools/ubench_stream
$U 65536 27648 2 64; $U 65536 27648 2 64 2; $U 65536 27648 3 64 2; $U 0 27648 2 64 2; $U 65536 27648 2 64 1
