// Scheme coefficient tables shared by the device kernels (expm_common.cuh)
// and the host-side drop-in (taylor_schemes.hpp / pade.hpp accessors in
// dropin_dense.cpp): one list of literals, the reference's doubles bit for
// bit (checked against the compiled reference by
// tests/test_oracle.py::test_device_coefficients_equal_reference).
#pragma once

namespace mexp_b200 {

// T8: closed forms in sqrt(177) with x3 = 2/3, as the reference rounds them
// once from long double (taylor_schemes.cpp:12-27); the hex literals are
// those doubles.
struct T8C {
    static constexpr double x1 = 0x1.bbdc940ef503ap-4;
    static constexpr double x2 = 0x1.bbdc940ef503ap-6;
    static constexpr double x3 = 0x1.5555555555555p-1;
    static constexpr double x4 = 0x1.17f11e296523cp-1;
    static constexpr double x5 = 0x1.49fc346242b21p-3;
    static constexpr double x6 = 0x1.cdbb2e2ed5250p-7;
    static constexpr double x7 = 0x1.14d4a1c010d67p-5;
    static constexpr double y0 = 1.0;
    static constexpr double y1 = 1.0;
    static constexpr double y2 = 0x1.157d04e6f24b6p-3;
};

}  // namespace mexp_b200

// T12 (paper eq. for the 4-product scheme; reference taylor_schemes.cpp:62-71):
// [i][j] multiplies {I, A, A2, A3}[i] in B_{j+1}.
#define MEXP_T12_TABLE { \
    {9.0198e-16, 5.31597895759871264183, 0.18188869982170434744, -2.0861320e-13}, \
    {0.46932117595418237389, 1.19926790417132231573, 0.05502798439925399070, \
     -0.13181061013830184015}, \
    {-0.20099424927047284052, 0.01179296240992997031, 0.09351590770535414968, \
     -0.02027855540589259079}, \
    {-0.04623946134063071740, 0.01108844528519167989, 0.00610700528898058230, \
     -0.00675951846863086359}, \
}

// T18 (reference taylor_schemes.cpp:73-85): A[i] multiplies {I,A,A2,A3}[i]
// in B1; B[j][r] multiplies {I,A,A2,A3,A6}[r] in B_{j+2}.
#define MEXP_T18A_TABLE {0.0, -0.100365581030144620, -0.0080292464824115696, \
                                 -0.0008921384980457299}
#define MEXP_T18B_TABLE { \
    {0.0, 0.39784974949964507614, 1.36783778460411719922, 0.49828962252538267755, \
     -0.0006378981945947233}, \
    {-10.967639605296206259, 1.68015813878906197182, 0.05717798464788655127, \
     -0.0069821012248805208, 0.00003349750170860705}, \
    {-0.0904316832390810561, -0.0676404519071381907, 0.06759613017704596460, \
     0.02955525704293155274, -0.0000139180257516060}, \
    {0.0, 0.0, -0.0923364619367118592, -0.0169364939002081717, -0.0000140086798182036}, \
}

// pade_coeffs(m).b (pade.cpp:34-48: exact integer ratios, rounded once via
// long double) as the compiled reference holds them, b_0..b_m for m = 1..13;
// checked bit for bit by tests/test_oracle.py::test_pade_coefficients.
#define MEXP_PADE_TABLE                                                               \
    {{1.0, 0x1.0000000000000p-1, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0}, \
     {1.0, 0x1.0000000000000p-1, 0x1.5555555555555p-4, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0}, \
     {1.0, 0x1.0000000000000p-1, 0x1.999999999999ap-4, 0x1.1111111111111p-7, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0}, \
     {1.0, 0x1.0000000000000p-1, 0x1.b6db6db6db6dbp-4, 0x1.8618618618618p-7, 0x1.3813813813814p-11, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0}, \
     {1.0, 0x1.0000000000000p-1, 0x1.c71c71c71c71cp-4, 0x1.c71c71c71c71cp-7, 0x1.0410410410410p-10, 0x1.1566abc011567p-15, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0}, \
     {1.0, 0x1.0000000000000p-1, 0x1.d1745d1745d17p-4, 0x1.f07c1f07c1f08p-7, 0x1.4afd6a052bf5bp-10, 0x1.08cabb37565e2p-14, 0x1.937e11175f095p-20, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0}, \
     {1.0, 0x1.0000000000000p-1, 0x1.d89d89d89d89ep-4, 0x1.0690690690690p-6, 0x1.7de952f2466a4p-10, 0x1.6ea28d118b474p-14, 0x1.b287c3a303e2bp-19, 0x1.f09b28ba4d955p-25, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0}, \
     {1.0, 0x1.0000000000000p-1, 0x1.ddddddddddddep-4, 0x1.1111111111111p-6, 0x1.a41a41a41a41ap-10, 0x1.c01c01c01c01cp-14, 0x1.45e5d2ba42ea0p-18, 0x1.29f6b20961c00p-23, 0x1.08db48ebe51c7p-29, 0.0, 0.0, 0.0, 0.0, 0.0}, \
     {1.0, 0x1.0000000000000p-1, 0x1.e1e1e1e1e1e1ep-4, 0x1.1919191919192p-6, 0x1.c1c1c1c1c1c1cp-10, 0x1.0101010101010p-13, 0x1.a5c001a5c001ap-18, 0x1.e20001e20001ep-23, 0x1.5e8ba44745d2dp-28, 0x1.f28db670be53bp-35, 0.0, 0.0, 0.0, 0.0}, \
     {1.0, 0x1.0000000000000p-1, 0x1.e50d79435e50dp-4, 0x1.1f7047dc11f70p-6, 0x1.d96da388960f5p-10, 0x1.1c0e9551f3a2dp-13, 0x1.f8fd7b3c5bcc1p-18, 0x1.49ca1c3c50d8ep-22, 0x1.306bcb4b5e520p-27, 0x1.68cb9b9bb2285p-33, 0x1.a3d5a71b92cd3p-40, 0.0, 0.0, 0.0}, \
     {1.0, 0x1.0000000000000p-1, 0x1.e79e79e79e79ep-4, 0x1.2492492492492p-6, 0x1.ecc07b301ecc0p-10, 0x1.3299e6401329ap-13, 0x1.2090d8b4c6bdcp-17, 0x1.9c3ca34b650f1p-22, 0x1.b7b825a5c1212p-27, 0x1.4f06351093257p-32, 0x1.49deba27f3581p-38, 0x1.3fdfbc45c52eap-45, 0.0, 0.0}, \
     {1.0, 0x1.0000000000000p-1, 0x1.e9bd37a6f4deap-4, 0x1.28cfc4a33f129p-6, 0x1.fcd1e360fe68fp-10, 0x1.45a50c670938fp-13, 0x1.3fee80f4f29acp-17, 0x1.e783d0b234bb0p-22, 0x1.1ec6024ab59b3p-26, 0x1.fdd1cb2f7bbe9p-32, 0x1.4648d3f56deaap-37, 0x1.0f328eed3d6fep-43, 0x1.bd0ac3296b624p-51, 0.0}, \
     {1.0, 0x1.0000000000000p-1, 0x1.eb851eb851eb8p-4, 0x1.2c5f92c5f92c6p-6, 0x1.0531b747fa105p-9, 0x1.55ed4d05c9af0p-13, 0x1.5b5ab7e55f2bap-17, 0x1.15e22cb77f562p-21, 0x1.5f02bf38a0d89p-26, 0x1.5aad6134c4c94p-31, 0x1.05070ff78b221p-36, 0x1.1cc1e2df80824p-42, 0x1.94fcfe65b1145p-49, 0x1.1cd3b01a822a6p-56} \
    }
