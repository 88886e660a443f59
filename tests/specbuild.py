"""Build product datatypes from flatten_oracle-style tuple specs."""


def build_product(spec, mp):
    k = spec[0]
    if k == "basic":
        return {1: mp.BYTE, 4: mp.INT32, 8: mp.INT64}[spec[1]]
    if k == "contiguous":
        return mp.type_contiguous(spec[1], build_product(spec[2], mp)).commit()
    if k == "vector":
        return mp.type_vector(spec[1], spec[2], spec[3], build_product(spec[4], mp)).commit()
    if k == "hvector":
        return mp.type_hvector(spec[1], spec[2], spec[3], build_product(spec[4], mp)).commit()
    if k == "indexed_block":
        return mp.type_indexed_block(spec[1], list(spec[2]), build_product(spec[3], mp)).commit()
    if k == "struct":
        return mp.type_create_struct(list(spec[1]), list(spec[2]),
                                     [build_product(c, mp) for c in spec[3]]).commit()
    if k == "subarray":
        return mp.type_create_subarray(list(spec[1]), list(spec[2]), list(spec[3]),
                                       build_product(spec[4], mp)).commit()
    if k == "resized":
        return mp.type_create_resized(build_product(spec[3], mp), spec[1], spec[2]).commit()
    if k == "indexed":
        return mp.type_indexed(list(spec[1]), list(spec[2]), build_product(spec[3], mp)).commit()
    raise ValueError(k)
