# decoupled table / entry rings: nibble tables (32 KB) leave room for a deeper entry ring
U=tools/ubench_stream
$U R 65536 27648 2 2 64; $U R 65536 27648 2 1 64
$U R 32768 27648 2 2 64; $U R 32768 27648 2 4 64; $U R 32768 27648 2 5 64; $U R 32768 27648 3 4 64
$U R 65536 13824 2 4 64
