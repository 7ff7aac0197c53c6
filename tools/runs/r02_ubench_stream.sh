# what bounds the staged plan's stream: tools/ubench_stream T E S phases [touch]
U=tools/ubench_stream
$U 65536 27648 2 64; $U 65536 27648 2 64 1
$U 0 27648 2 64; $U 65536 0 2 64
$U 0 27648 4 64; $U 0 27648 6 64; $U 0 13824 8 128
$U 32768 27648 2 64; $U 32768 27648 3 64
$U 16384 27648 2 64; $U 16384 27648 4 64
$U 32768 13824 4 128; $U 32768 13824 6 128
$U 65536 27648 2 64 1
